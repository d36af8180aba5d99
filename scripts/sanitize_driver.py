"""Smoke-sized invocations of every libtwb200 kernel, each checked against the C oracle or
numpy, for compute-sanitizer (scripts/sanitize.sh; tests/test_sanitizer.py):

  k_sim<false>  latency variant, blob staged by TMA (8 configs, Timekeeper grid on, audit dump)
  k_seg_plan, k_sim_seg, k_seg_tk, k_sim_join  busy-period segments (clean joins, overruns,
                forced overflows and serial re-runs in the join)
  k_sim<true>   throughput variant (forced by a 367 KB predictor blob that cannot be staged)
  k_predict_features<true/false>, k_predict_batches<true/false> (mbarrier producer/consumer pipeline)
  k_tk_replay, k_tk_resolve_rows, k_metrics, k_generate_poisson, k_predict_single,
  k_predict_service (persistent polling warp; closed before any device-wide sync)
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as orc  # noqa: E402
from paper_2601_00397_b200 import _lib, presets  # noqa: E402
from paper_2601_00397_b200.predictor import BatchComposition, DecodeSlot, PredictorSet, PrefillChunk, TablePredictor  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep  # noqa: E402
from paper_2601_00397_b200.timekeeper import OpStream, replay_many, resolve_round  # noqa: E402
from paper_2601_00397_b200.workload import WorkloadSpec, generate_device, poisson_arrays  # noqa: E402

which = set(sys.argv[1:]) or {"sim", "seg", "simtput", "bulk", "tk", "metrics", "wl", "single", "service"}
rng = np.random.default_rng(0)


def check_sim(sub, dev):
    d = DeviceSweep(sub.pset, sub.workloads, sub.cfgs, per_request=True, audit=[0])
    d.run()
    torch.cuda.synchronize()
    got = d.fetch()
    want, _, first, finish = orc.sim_many(sub.pset.blob, sub.cfgs, sub.workloads.wl_off, sub.workloads.offset_ns,
                                          sub.workloads.prompt, sub.workloads.output, per_request=True)
    for f in ("status", "final_now_ns", "steps", "events", "digest", "tk_seq", "tk_offset_ns", "tk_wall_ns"):
        assert np.array_equal(got.results[f], want[f]), f
    assert np.array_equal(got.first_ns, first[: len(got.first_ns)]) and np.array_equal(got.finish_ns, finish[: len(got.finish_ns)])
    return d, got


if "sim" in which or "metrics" in which:
    sw = presets.sweep_1024(n_requests=60)
    sub = sw.subset(np.arange(0, len(sw), 128))
    d, got = check_sim(sub, "cuda")
    print("k_sim latency ok", _lib.last_sim_launch()["variant"])
    if "metrics" in which:
        d.run_metrics()
        m = d.fetch_metrics()
        w = sub.workloads
        for k in range(len(sub)):
            lo, hi = int(w.wl_off[sub.cfgs[k]["workload_id"]]), int(w.wl_off[sub.cfgs[k]["workload_id"] + 1])
            rb = int(d.req_base[k])
            want_m = orc.metrics(w.offset_ns[lo:hi], w.output[lo:hi], got.first_ns[rb: rb + hi - lo],
                                 got.finish_ns[rb: rb + hi - lo], int(sub.cfgs[k]["epoch_ns"]))
            assert m[k].tobytes() == want_m.tobytes()
        print("k_metrics ok")

if "seg" in which:
    import os

    def check_seg(sub, env):
        os.environ.update(env)
        try:
            d = DeviceSweep(sub.pset, sub.workloads, sub.cfgs, per_request=True)
            d.run()
            torch.cuda.synchronize()
            got = d.fetch()
        finally:
            for k in env:
                os.environ.pop(k, None)
        assert _lib.last_sim_launch()["variant"] == "segments"
        want, _, first, finish = orc.sim_many(sub.pset.blob, sub.cfgs, sub.workloads.wl_off, sub.workloads.offset_ns,
                                              sub.workloads.prompt, sub.workloads.output, per_request=True)
        for f in ("status", "final_now_ns", "steps", "events", "digest", "tk_seq", "tk_offset_ns", "tk_wall_ns"):
            assert np.array_equal(got.results[f], want[f]), f
        assert np.array_equal(got.first_ns, first[: len(got.first_ns)])
        assert np.array_equal(got.finish_ns, finish[: len(got.finish_ns)])
        # hand the (large) segment scratch back at once, so later allocations are not carved
        # out of its cached block (memcheck --leak-check would report the block as leaked)
        del d, got
        torch.cuda.empty_cache()

    sw = presets.sweep_1024(n_requests=160)
    sub = sw.subset(np.arange(0, len(sw), 128))
    check_seg(sub, {"TWB_SIM_SEG_W": "8"})
    check_seg(sub, {"TWB_SIM_SEG_W": "8", "TWB_SIM_SEG_CAPDIV": "1000"})  # every segment out of room
    heavy = presets.single("heavy", "70b", 4, 2, 400, 4)  # long busy periods: overruns
    check_seg(heavy, {"TWB_SIM_SEG_W": "25"})
    print("k_seg_plan / k_sim_seg / k_seg_tk / k_sim_join ok")

big = None
if "simtput" in which or "bulk" in which:
    preds = []
    for _ in range(48):
        pax = np.unique(np.concatenate([[0], rng.integers(1, 9000, 23)]))
        dax = np.unique(np.concatenate([[0], rng.integers(1, 600, 23)]))
        rows = {(int(p), int(dd)): int(800 + 9 * p + 35 * dd + rng.integers(0, 50))
                for p in pax for dd in dax if (p, dd) != (0, 0)}
        preds.append(TablePredictor(rows, allow_extrapolation=True))
    big = PredictorSet(preds)
if "simtput" in which:
    sw = presets.sweep_1024(n_requests=40)
    sub = sw.subset(np.arange(0, len(sw), 256))
    sub.pset = big
    sub.cfgs["pred_id"] = np.arange(len(sub)) % 48
    check_sim(sub, "cuda")
    assert _lib.last_sim_launch()["variant"] == "throughput"
    print("k_sim throughput ok")

if "bulk" in which:
    for pset in (presets.calibration_set(), big):
        n = 20_003
        P = rng.integers(0, 9000, n).astype(np.int32)
        D = rng.integers(0, 600, n).astype(np.int32)
        C = rng.integers(0, 10**5, n).astype(np.int64)
        I = rng.integers(0, len(pset.predictors), n).astype(np.int32)
        assert np.array_equal(pset.predict_features(P, D, C, I), orc.predict_many(pset.blob, P, D, C, I))
        counts = rng.integers(0, 9, 7001)
        off = np.zeros(len(counts) + 1, np.int64)
        np.cumsum(counts, out=off[1:])
        tok = np.where(rng.random(int(off[-1])) < 0.7, -1, rng.integers(1, 700, int(off[-1]))).astype(np.int32)
        ctx = rng.integers(0, 3000, int(off[-1])).astype(np.int32)
        ids = rng.integers(0, len(pset.predictors), len(counts)).astype(np.int32)
        ns, feat = pset.predict_csr(off, tok, ctx, ids, return_features=True)
        assert np.array_equal(feat, orc.extract_features(off, tok, ctx))
    print("k_predict_features / k_predict_batches ok (staged and global blob)")

if "tk" in which:
    h = OpStream(cooldown_ns=500_000)
    acts = [h.register_actor() for _ in range(17)]
    h.seal()
    for k in range(5):
        for i, a in enumerate(acts):
            h.jump(a, 1_000_000_000 + (k + 1) * 10_000_000 + i * 1000)
    r = replay_many([h, h])
    assert r.broadcast_sequence(0) == r.broadcast_sequence(1) and len(r.broadcast_sequence(0)) == 5
    A, C = 17, 3000
    pend = rng.integers(1, 10**12, C * A).astype(np.int64)
    elig = np.full(C, (1 << A) - 1, np.uint32)
    st = [pend, rng.integers(0, 10**9, C), np.zeros(C, np.int64), rng.integers(0, 10**12, C), np.full(C, -(1 << 63))]
    st = [np.asarray(x, np.int64) for x in st]
    cpu = [x.copy() for x in st]
    want = orc.tk_resolve(cpu[0], elig, A, 500_000, cpu[1], cpu[2], cpu[3], cpu[4])
    dv = [torch.from_numpy(x.copy()).cuda() for x in st]
    got = resolve_round(dv[0], torch.from_numpy(elig.view(np.int32)).cuda(), A, 500_000, *dv[1:])
    assert np.array_equal(got.cpu().numpy(), want)
    print("k_tk_replay / k_tk_resolve_rows ok")

if "wl" in which:
    spec = WorkloadSpec.from_doc({"source": "poisson", "qps": 8, "seed": 5, "num_requests": 300,
                                  "prompt_tokens": {"kind": "uniform", "low": 64, "high": 2048},
                                  "output_tokens": {"kind": "uniform", "low": 16, "high": 256}})
    gen = generate_device([spec, spec])
    for a_, b_ in zip(gen.workload(1), poisson_arrays(spec)):
        assert np.array_equal(a_, b_)
    print("k_generate_poisson ok")

batches = [BatchComposition(tuple(PrefillChunk(f"p{i}", int(rng.integers(1, 900)), 0) for i in range(int(rng.integers(0, 3)))),
                            tuple(DecodeSlot(f"d{i}", 100) for i in range(int(rng.integers(0, 40))))) for _ in range(40)]
pset = presets.calibration_set()
ids = rng.integers(0, len(pset.predictors), len(batches)).astype(np.int32)
if "single" in which or "service" in which:
    want = pset.predict_batches(batches, ids)
if "single" in which:
    got = [pset.predictors[int(k)].predict(b) if not b.is_empty() else -1 for b, k in zip(batches, ids)]
    assert all(g == w for g, w in zip(got, want) if w >= 0)
    print("k_predict_single ok")
if "service" in which:
    sv = pset.service()
    try:
        got = [sv.predict_one(b, int(k)) for b, k in zip(batches, ids)]
    finally:
        sv.close()
    assert np.array_equal(np.asarray(got, np.int64), want)
    print("k_predict_service ok")
torch.cuda.synchronize()
print(f"sanitize driver done: {_lib.launch_count()} launches")
# hand torch's cached device and pinned blocks back so --leak-check reports only what the
# engine itself would leak
import gc  # noqa: E402

for name in list(globals()):
    if not name.startswith("_") and name not in ("gc", "torch", "which", "sys", "presets"):
        globals().pop(name, None)
presets._PSET = None  # the cached calibration set holds its device blob
gc.collect()
torch.cuda.empty_cache()
if hasattr(torch._C, "_host_emptyCache"):
    torch._C._host_emptyCache()
