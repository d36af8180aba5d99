#!/usr/bin/env python
"""Benchmark: emulated virtual-seconds per wall-second over a config sweep on B200.

Metric (BASELINE.json): "emulated virtual-sec/wall-sec over config sweep; batch
predictions/sec @1/2/4/8 GPU". One step = one pass of the hot path over one batch
of synthetic input = the full event loop (oracle.simulate semantics + Timekeeper
actor grid) of every config in the sweep, in one persistent tw_sim_many launch per GPU.

Workload (the same at every N, strong scaling): BASELINE config 5, the 65,536-config
sweep (the config-4 grid x {Llama-3-8B, 70B} tables x 32 Poisson workload seeds),
sharded over the N ranks by a cost-model LPT partition; at N > 1 the records of all
ranks are merged with one NCCL all-gather inside the e2e window. At N = 1 the line also
carries BASELINE config 4 (the 1,024-config sweep on one B200) as `config4`, and the
projected N = 2/4/8 step times (each rank's shard timed alone on this GPU).
`--sweep 1024` makes config 4 the headline instead (weak scaling, seed 1 + rank).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

value  = sum over all configs of virtual span / max-over-ranks device time per step
e2e    = the same through the public host API (pinned host inputs -> H2D -> kernel ->
         result records and per-request stamps in pinned host memory -> at N > 1 the
         NCCL gather + merge of all records), timed with CUDA events, max over ranks
roofline / predictor_roofline / cpu_baseline: see DESIGN.md §Measurement.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2, written between timed iterations


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--sweep", choices=("1024", "65536"), default="65536")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-projection", action="store_true", help="skip the per-shard strong-scaling projection")
    ap.add_argument("--no-config4", action="store_true", help="skip the config-4 block at N = 1")
    ap.add_argument("--no-configs13", action="store_true", help="skip the BASELINE configs 1-3 block at N = 1")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--share-device", action="store_true",
                    help="all ranks on cuda:0 with gloo collectives: a one-GPU dry run of the multi-rank path")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def build_workload(args, world, rank):
    from paper_2601_00397_b200 import presets
    from paper_2601_00397_b200.distributed import partition
    from paper_2601_00397_b200.sweep import estimate_cost

    if args.sweep == "1024":
        sw = presets.sweep_1024(model="8b", seed=1 + rank)
        config = {"workload": "BASELINE config 4: 1,024-config sweep per GPU (weak scaling)",
                  "model": "Llama-3-8B calibration tables (synthetic)", "configs_per_gpu": len(sw),
                  "requests_per_config": 1000, "qps": 8, "workload_seed": f"1 + rank",
                  "grid": "mbt{1024..8192} x chunk{128..1024} x max_running{32..256} x (TP,PP) x 8 x policy x 2",
                  "timekeeper": "dispatcher + TP*PP workers, cooldown 500us", "parallelism": f"configs sharded, dp{world}",
                  "l2": "flushed (512 MiB write) between timed iterations"}
        sw.global_ids = np.arange(len(sw), dtype=np.int64) + rank * len(sw)
        sw.n_global = len(sw) * world
        return sw, config, "weak"
    full = presets.sweep_65536()
    shards = partition(estimate_cost(full.pset, full.cfgs, full.workloads), world)
    sw = full.subset(shards[rank])
    sw.global_ids = shards[rank]
    sw.n_global = len(full)
    config = {"workload": "BASELINE config 5: 65,536-config sweep sharded over GPUs (strong scaling)",
              "model": "Llama-3-8B/70B calibration tables (synthetic)", "configs_total": len(full),
              "configs_rank0": len(sw), "requests_per_config": 1000, "qps": 8, "workload_seeds": "1..32",
              "grid": "mbt{1024..8192} x chunk{128..1024} x max_running{32..256} x (TP,PP) x 8 x policy x 2",
              "timekeeper": "dispatcher + TP*PP workers, cooldown 500us",
              "parallelism": f"configs sharded by cost-model LPT, dp{world}",
              "l2": "flushed (512 MiB write) between timed iterations"}
    return sw, config, "strong"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def n_req_e2e(host) -> int:
    return int(host.req_base[-1])


def flush_l2(buf):
    buf.fill_(1)  # a plain write larger than L2


def time_kernel_steps(run, steps, warmup, flush_buf, stream):
    """Per-step CUDA-event durations of `run()` on `stream`, L2 flushed before each."""
    import torch

    for _ in range(warmup):
        flush_l2(flush_buf)
        run()
    torch.cuda.synchronize()
    durs = []
    for _ in range(steps):
        flush_l2(flush_buf)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run()
        b.record(stream)
        b.synchronize()
        durs.append(a.elapsed_time(b))
    return durs


def measured_traffic(kernel: str):
    """DRAM bytes per launch from the committed ncu capture (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh)[kernel]["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def measured_issue(kernel: str):
    """What bounds a latency-bound kernel, from the committed ncu capture
    (profiles/traffic.json): issue-slot use and the dominant stall reasons."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            entry = json.load(fh)[kernel]
    except (OSError, KeyError, ValueError):
        return None
    if "issue" in entry:
        return entry["issue"]
    return {k: v for k, v in entry.items() if k != "dram_bytes_per_launch"}


def predictor_roofline(device, peak_gbs):
    """Bulk predictor kernel (tw_predict_features) at 2^27 queries: achieved GB/s vs HBM peak."""
    import torch

    from paper_2601_00397_b200 import _lib, presets
    from paper_2601_00397_b200._device import stream_handle

    pset = presets.calibration_set()
    n = 1 << 27
    g = torch.Generator(device=device).manual_seed(0)
    P = torch.randint(0, 8192, (n,), dtype=torch.int32, device=device, generator=g)
    D = torch.randint(0, 257, (n,), dtype=torch.int32, device=device, generator=g)
    C = torch.randint(0, 600_000, (n,), dtype=torch.int64, device=device, generator=g)
    I = torch.randint(0, 16, (n,), dtype=torch.int32, device=device, generator=g)
    out = torch.empty(n, dtype=torch.int64, device=device)
    blob = pset.device_blob(device)
    lib = _lib.load()
    s = torch.cuda.current_stream()

    def run():
        _lib.check(lib.tw_predict_features(blob.data_ptr(), pset.nbytes, P.data_ptr(), D.data_ptr(), C.data_ptr(),
                                           I.data_ptr(), n, out.data_ptr(), stream_handle(s)), "predict")

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    durs = []
    for _ in range(10):  # inputs (3.7 GB) far exceed L2: no flush needed
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        run()
        b.record(s)
        b.synchronize()
        durs.append(a.elapsed_time(b))
    ms = statistics.median(durs)
    bytes_per = 4 + 4 + 8 + 4 + 8  # P, D, C, desc_id in; ns out
    gbs = n * bytes_per / (ms / 1e3) / 1e9
    del P, D, C, I, out
    return {"kernel": "k_predict_features", "bound": "hbm", "achieved": round(gbs, 1), "peak": peak_gbs,
            "unit": "GB/s", "frac": round(gbs / peak_gbs, 4), "bytes_per_prediction": bytes_per,
            "predictions_per_launch": n, "ms_per_launch": round(ms, 4),
            "predictions_per_s": round(n / (ms / 1e3), 1), "traffic": measured_traffic("k_predict_features"),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, burst)"}


def extraction_roofline(device, peak_gbs, nb: int = 1 << 25):
    """Fused batch-feature extraction + prediction (tw_predict_batches) over 2^25 CSR
    batches of 1-8 slots (70% decode slots), Table models; inputs far exceed L2. Two
    launches of the same batches, each with its own algorithmic bytes:

    * headline, features out (north-star kernel 1's product plus the durations): 8 offset +
      4 descriptor id + 8 ns + 24 features {P, D, C} per batch and 8 (token, context) per
      slot, every byte read or written by the kernel;
    * `predictions_only` (no features): the calibration set's models never read
      total_context, so the kernel does not read slot_ctx: 20 B per batch + 4 per slot.
      (Round 1 counted the context slots here too: 20 + 8 per slot.)"""
    import torch

    from paper_2601_00397_b200 import _lib, presets
    from paper_2601_00397_b200._device import stream_handle

    pset = presets.calibration_set()
    g = torch.Generator(device=device).manual_seed(1)
    counts = torch.randint(1, 9, (nb,), device=device, generator=g)
    off = torch.zeros(nb + 1, dtype=torch.int64, device=device)
    off[1:] = torch.cumsum(counts, 0)
    ns = int(off[-1].item())
    ns_pad = (ns + 3) // 4 * 4
    tok = torch.randint(1, 700, (ns_pad,), dtype=torch.int32, device=device, generator=g)
    tok[torch.rand(ns_pad, device=device, generator=g) < 0.7] = -1
    ctx = torch.randint(0, 3000, (ns_pad,), dtype=torch.int32, device=device, generator=g)
    ids = torch.randint(0, 16, (nb,), dtype=torch.int32, device=device, generator=g)
    out = torch.empty(nb, dtype=torch.int64, device=device)
    feat = torch.empty(nb, 3, dtype=torch.int64, device=device)
    blob = pset.device_blob(device)
    lib = _lib.load()
    s = torch.cuda.current_stream()

    def timed(with_feat):
        fp = feat.data_ptr() if with_feat else None

        def run():
            _lib.check(lib.tw_predict_batches(blob.data_ptr(), pset.nbytes, off.data_ptr(), tok.data_ptr(),
                                              ctx.data_ptr(), ids.data_ptr(), nb, fp, out.data_ptr(),
                                              stream_handle(s)), "extract")

        for _ in range(3):
            run()
        torch.cuda.synchronize()
        durs = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            run()
            b.record(s)
            b.synchronize()
            durs.append(a.elapsed_time(b))
        return statistics.median(durs)

    ms_f = timed(True)
    ms_p = timed(False)
    alg_f = nb * (8 + 4 + 8 + 24) + ns * 8
    alg_p = nb * (8 + 4 + 8) + ns * 4
    gbs_f = alg_f / (ms_f / 1e3) / 1e9
    gbs_p = alg_p / (ms_p / 1e3) / 1e9
    del off, tok, ctx, ids, out, feat
    return {"kernel": "k_predict_batches", "bound": "hbm", "achieved": round(gbs_f, 1), "peak": peak_gbs,
            "unit": "GB/s", "frac": round(gbs_f / peak_gbs, 4), "outputs": "features {P, D, C} + ns per batch",
            "batches_per_launch": nb, "slots_per_launch": ns, "bytes_per_batch": round(alg_f / nb, 2),
            "ms_per_launch": round(ms_f, 4), "batches_per_s": round(nb / (ms_f / 1e3), 1),
            "traffic": measured_traffic("k_predict_batches"),
            "predictions_only": {"achieved": round(gbs_p, 1), "frac": round(gbs_p / peak_gbs, 4),
                                 "bytes_per_batch": round(alg_p / nb, 2), "ms_per_launch": round(ms_p, 4),
                                 "batches_per_s": round(nb / (ms_p / 1e3), 1),
                                 "note": "no features requested; Table models never read slot_ctx"}}


def timekeeper_roofline(device, peak_gbs, A: int = 17):
    """Bulk Timekeeper min-advance (tw_tk_resolve): one BarrierCore round for C
    independent Timekeepers of A actors (dispatcher + TP8 x PP2 workers), every actor
    eligible with a pending target, so every round resolves. Reported as
    latency per advance step at C = 65,536 (the config-5 sweep) and as GB/s at C = 2^21
    (algorithmic bytes per Timekeeper: 8A pending + 4 mask + 32 state read, 8A pending
    clear + 32 state + 1 flag written). Pending targets are restored before each round
    (not timed)."""
    import torch

    from paper_2601_00397_b200 import _lib
    from paper_2601_00397_b200._device import stream_handle

    lib = _lib.load()
    s = torch.cuda.current_stream()
    out = {"kernel": "k_tk_resolve_rows", "bound": "hbm", "actors": A, "peak": peak_gbs, "unit": "GB/s"}
    for C in (65536, 1 << 21):
        g = torch.Generator(device=device).manual_seed(C)
        base = 1_790_000_000_000_000_000
        pend0 = base + torch.randint(1, 10**9, (C * A,), dtype=torch.int64, device=device, generator=g)
        pending = pend0.clone()
        elig = torch.full((C,), (1 << A) - 1, dtype=torch.int32, device=device)
        offset = torch.zeros(C, dtype=torch.int64, device=device)
        seq = torch.zeros(C, dtype=torch.int64, device=device)
        wall = torch.full((C,), base, dtype=torch.int64, device=device)
        last = torch.full((C,), base - 1_000_000, dtype=torch.int64, device=device)
        bc = torch.empty(C, dtype=torch.int8, device=device)
        durs = []
        for i in range(13):
            pending.copy_(pend0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            _lib.check(lib.tw_tk_resolve(pending.data_ptr(), elig.data_ptr(), C, A, 500_000, offset.data_ptr(),
                                         seq.data_ptr(), wall.data_ptr(), last.data_ptr(), bc.data_ptr(),
                                         stream_handle(s)), "tk_resolve")
            b.record(s)
            b.synchronize()
            if i >= 3:
                durs.append(a.elapsed_time(b))
        assert bool((bc >= 0).all())  # every round resolves (|pending| == eligible)
        ms = statistics.median(durs)
        alg = C * (16 * A + 4 + 32 + 33)
        key = "config5" if C == 65536 else "bulk"
        out[key] = {"timekeepers": C, "us_per_advance_step": round(ms * 1e3, 2),
                    "achieved": round(alg / (ms / 1e3) / 1e9, 1)}
        del pend0, pending, elig, offset, seq, wall, last, bc
    out["achieved"] = out["bulk"]["achieved"]
    out["frac"] = round(out["achieved"] / peak_gbs, 4)
    out["traffic"] = measured_traffic("k_tk_resolve")
    return out


def workload_generation(device, n_wl: int = 65536, n_req: int = 1000):
    """tw_generate_poisson: config-5-shaped workloads (qps 8, prompt U[64, 2048], output
    U[16, 256], 1,000 requests) for n_wl distinct seeds in one launch, against the
    reference's host generator (numpy, one process) timed on a sample."""
    import torch

    from paper_2601_00397_b200 import _lib
    from paper_2601_00397_b200._device import stream_handle
    from paper_2601_00397_b200.workload import WorkloadSpec, poisson_arrays, wl_specs

    doc = {"source": "poisson", "qps": 8, "num_requests": n_req,
           "prompt_tokens": {"kind": "uniform", "low": 64, "high": 2048},
           "output_tokens": {"kind": "uniform", "low": 16, "high": 256}}
    specs = [WorkloadSpec.from_doc({**doc, "seed": 1000 + i}) for i in range(n_wl)]
    sp = torch.from_numpy(wl_specs(specs).view(np.uint8).copy()).to(device)
    off = torch.arange(n_wl + 1, dtype=torch.int64, device=device) * n_req
    ts = torch.empty(n_wl * n_req, dtype=torch.int64, device=device)
    pr = torch.empty(n_wl * n_req, dtype=torch.int32, device=device)
    op = torch.empty(n_wl * n_req, dtype=torch.int32, device=device)
    st = torch.empty(n_wl, dtype=torch.int32, device=device)
    lib = _lib.load()
    s = torch.cuda.current_stream()

    def run():
        _lib.check(lib.tw_generate_poisson(sp.data_ptr(), n_wl, off.data_ptr(), ts.data_ptr(), pr.data_ptr(),
                                           op.data_ptr(), st.data_ptr(), stream_handle(s)), "generate")

    run()
    torch.cuda.synchronize()
    durs = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        run()
        b.record(s)
        b.synchronize()
        durs.append(a.elapsed_time(b))
    ms = statistics.median(durs)
    ok = bool((st == 0).all()) and np.array_equal(ts[:n_req].cpu().numpy(), poisson_arrays(specs[0])[0])
    t0 = time.perf_counter()
    k = 0
    while time.perf_counter() - t0 < 2.0:
        poisson_arrays(specs[k % n_wl])
        k += 1
    host_rps = k * n_req / (time.perf_counter() - t0)
    del ts, pr, op
    return {"kernel": "k_generate_poisson", "workloads": n_wl, "requests": n_wl * n_req, "ms_per_launch": round(ms, 3),
            "requests_per_s": round(n_wl * n_req / (ms / 1e3), 1), "host_numpy_requests_per_s_one_core": round(host_rps, 1),
            "matches_host": ok, "bound": "latency",
            "note": "one thread per workload runs its sequential PCG64 stream; outputs staged per warp and "
                    "written as coalesced rows"}


def metrics_roofline(dev, args, flush, stream, peak_gbs):
    """tw_metrics_many over the sweep's stamps: every config's
    RunReport.summary() numbers. Algorithmic bytes: first + finish stamps (16 B),
    arrival offset (8 B) and output count (4 B) per request, 160 B out per config."""
    durs = time_kernel_steps(dev.run_metrics, args.steps, args.warmup, flush, stream)
    ms = sum(durs) / len(durs)
    m = dev.fetch_metrics()
    n_req = int(dev.req_base[-1])
    alg = 28 * n_req + 160 * dev.n_cfg
    gbs = alg / (ms / 1e3) / 1e9
    return {"kernel": "k_metrics", "bound": "latency", "achieved": round(gbs, 1), "peak": peak_gbs, "unit": "GB/s",
            "frac": round(gbs / peak_gbs, 4), "traffic": measured_traffic("k_metrics"), "ms_per_launch": round(ms, 4),
            "configs_per_s": round(dev.n_cfg / (ms / 1e3), 1), "requests_per_s": round(n_req / (ms / 1e3), 1),
            "all_ok": bool((m["status"] == 0).all()), "algorithmic_bytes_per_launch": int(alg),
            "note": "one CTA per config: radix selection of three nearest ranks per metric and a serial "
                    "CPython-order compensated TPOT sum; HBM fraction shown for reference only"}


def cpu_baseline(sw, budget_s: float, n_threads: int):
    """The C oracle port over a stratified sample of the same sweep, all host threads."""
    from oracle import oracle as orc

    n = len(sw)
    take = max(1, min(n, 8 * n_threads))
    t_est = None
    while True:
        ids = np.linspace(0, n - 1, take).astype(np.int64)
        sub = sw.subset(ids)
        t0 = time.perf_counter()
        res, *_ = orc.sim_many(sub.pset.blob, sub.cfgs, sub.workloads.wl_off, sub.workloads.offset_ns,
                               sub.workloads.prompt, sub.workloads.output, n_threads=n_threads)
        dt = time.perf_counter() - t0
        if dt >= 0.5 * budget_s / 4 or take >= n:
            t_est = dt
            break
        take = min(n, int(take * max(2.0, (budget_s / 4) / max(dt, 1e-3))))
    vsec = float(res["final_now_ns"].astype(np.float64).sum()) / 1e9
    steps = int(res["steps"].sum())
    return {
        "value": round(vsec / t_est, 1), "unit": "virtual-s/wall-s", "cores": n_threads, "kind": "port",
        "sample": f"{take} of {n} configs (evenly spaced), C oracle (oracle/twb_oracle.c) on {n_threads} host threads",
        "steps_per_s": round(steps / t_est, 1), "seconds": round(t_est, 3),
    }


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _ref_simulate_one(job):
    """One config through the UNMODIFIED reference (baseline/_ref: timewarp.oracle.simulate
    with TablePredictor.from_csv, pkg/src/timewarp/oracle.py:49-114): virtual span, steps
    (= predict calls) and the final timestamp, for the Python CPU baseline."""
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from timewarp import oracle as ref_oracle
    from timewarp.engine import EngineConfig as RefEngineConfig
    from timewarp.engine import SchedulingPolicy as RefPolicy
    from timewarp.predictor import TablePredictor as RefTable
    from timewarp.workload import Arrival as RefArrival

    ts, prompt, output, eng, csv, epoch = job
    arrivals = [RefArrival(f"r{i}", int(t), int(p), int(o)) for i, (t, p, o) in enumerate(zip(ts, prompt, output))]
    cfg = RefEngineConfig(chunk_size=eng[0], policy=RefPolicy("mixed" if eng[7] == 0 else "prefill_prioritized"),
                          max_batch_tokens=eng[1], max_running=eng[2], kv_block_tokens=eng[3],
                          kv_capacity_blocks=eng[4], workers_per_replica=eng[5], pp_stages=eng[6])
    pred = RefTable.from_csv(csv, allow_extrapolation=True)
    calls = [0]
    inner = pred.predict

    def counting(batch, hw=None):
        calls[0] += 1
        return inner(batch, hw)

    pred.predict = counting
    events = ref_oracle.simulate(arrivals, cfg, pred, epoch_ns=epoch)
    last = max(e["virtual_ts_ns"] for e in events if e["kind"] == "FINISHED")
    return last - epoch, calls[0], last


def _ref_jobs(sw, ids):
    from paper_2601_00397_b200 import calibration

    grid = [(m, tp, pp) for m in calibration.MODELS for tp, pp in calibration.TP_PP_GRID]
    wl = sw.workloads
    jobs = []
    for c in ids:
        cf = sw.cfgs[c]
        lo, hi = int(wl.wl_off[cf["workload_id"]]), int(wl.wl_off[cf["workload_id"] + 1])
        eng = tuple(int(cf[k]) for k in ("chunk_size", "max_batch_tokens", "max_running", "kv_block_tokens",
                                           "kv_capacity_blocks", "workers_per_replica", "pp_stages", "policy"))
        jobs.append((wl.offset_ns[lo:hi].tolist(), wl.prompt[lo:hi].tolist(), wl.output[lo:hi].tolist(), eng,
                     calibration.csv_path(*grid[int(cf["pred_id"])]), int(cf["epoch_ns"])))
    return jobs


def cpu_baseline_python(sw, device_results, n_sample: int = 0):
    """SURVEY §8d's CPU path: multiprocessing.Pool(os.cpu_count()) over the unmodified
    reference's oracle.simulate (baseline/_ref) on an evenly spaced sample of the sweep
    (both models), wall-clock timed; each config's span and step count are also checked
    against this engine's device records."""
    import multiprocessing as mp

    if not os.path.isdir(os.path.join(REF_DIR, "timewarp")):
        return {"unavailable": "baseline/_ref has no timewarp package"}
    n = len(sw)
    procs = os.cpu_count() or 1
    ids = np.linspace(0, n - 1, min(n, n_sample or max(64, 8 * procs))).astype(np.int64)
    jobs = _ref_jobs(sw, ids)
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        out = pool.map(_ref_simulate_one, jobs, chunksize=1)
    dt = time.perf_counter() - t0
    span = np.array([o[0] for o in out], np.float64)
    steps = np.array([o[1] for o in out], np.int64)
    agree = bool(np.array_equal(steps, device_results["steps"][ids]) and
                 np.array_equal(np.array([o[2] for o in out], np.int64), device_results["final_now_ns"][ids]))
    return {"value": round(float(span.sum()) / 1e9 / dt, 2), "unit": "virtual-s/wall-s", "cores": procs,
            "kind": "reference",
            "sample": f"{len(ids)} of {n} configs (evenly spaced, both models), unmodified reference "
                      f"timewarp.oracle.simulate + TablePredictor.from_csv (baseline/_ref), Pool({procs})",
            "steps_per_s": round(float(steps.sum()) / dt, 1), "seconds": round(dt, 3),
            "matches_device_records": agree}


def configs_1_3(device):
    """BASELINE configs 1-3 (single configurations) on the GPU (one tw_sim_many
    launch each, CUDA events), beside the C port on one host thread and the unmodified
    Python reference (one process)."""
    import torch

    from oracle import oracle as orc
    from paper_2601_00397_b200 import presets
    from paper_2601_00397_b200.sweep import DeviceSweep

    out = {}
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=device)
    for name, mk in (("config1", presets.config1), ("config2", presets.config2), ("config3", presets.config3)):
        sw = mk()
        d = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, device=device, per_request=True)
        durs = time_kernel_steps(d.run, 5, 2, flush, torch.cuda.current_stream(device))
        ms = sum(durs) / len(durs)
        r = d.fetch().results
        with _Env(TWB_SIM_SEG=0):  # the serial loop (one warp), for comparison
            serial_ms = time_alone(sw, device)
        stats = seg_stats(sw, device)
        vs = float(r["final_now_ns"][0] - sw.cfgs["epoch_ns"][0]) / 1e9
        t0 = time.perf_counter()
        cres, *_ = orc.sim_many(sw.pset.blob, sw.cfgs, sw.workloads.wl_off, sw.workloads.offset_ns,
                                sw.workloads.prompt, sw.workloads.output, n_threads=1)
        c_s = time.perf_counter() - t0
        rec = {"label": sw.configs[0].label, "requests": int(sw.workloads.sizes()[0]), "steps": int(r["steps"][0]),
               "virtual_s": round(vs, 3), "gpu_ms": round(ms, 4), "gpu_virtual_s_per_wall_s": round(vs / (ms / 1e3), 1),
               "gpu_serial_loop_ms": round(serial_ms, 4), "segments": stats,
               "c_port_one_thread_ms": round(c_s * 1e3, 2), "c_port_matches": bool((cres == r).all())}
        if os.path.isdir(os.path.join(REF_DIR, "timewarp")):
            t0 = time.perf_counter()
            span, calls, last = _ref_simulate_one(_ref_jobs(sw, [0])[0])
            py_s = time.perf_counter() - t0
            rec |= {"python_reference_ms": round(py_s * 1e3, 1),
                    "python_reference_virtual_s_per_wall_s": round(span / 1e9 / py_s, 1),
                    "python_reference_matches": bool(calls == int(r["steps"][0]) and last == int(r["final_now_ns"][0]))}
        out[name] = rec
        del d
    return out


def run_reference(args):
    """--impl reference: the CPU implementation (C oracle port; the reference is pure Python
    and has no compiled path) on this box's host cores, same metric/config."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    sw, config, scaling = build_workload(args, 1, 0)
    from oracle import oracle as orc

    threads = os.cpu_count() or 1
    n = len(sw)
    # each step: an evenly spaced sample of the sweep sized to ~1/(K+W) of a ~3 min budget
    ids_all = np.arange(n)
    sample = max(threads, min(n, 4 * threads))
    vals, preds = [], []
    for i in range(args.warmup + args.steps):
        ids = ids_all[(np.arange(sample) * (n // sample) + i) % n]
        sub = sw.subset(ids)
        t0 = time.perf_counter()
        res, *_ = orc.sim_many(sub.pset.blob, sub.cfgs, sub.workloads.wl_off, sub.workloads.offset_ns,
                               sub.workloads.prompt, sub.workloads.output, n_threads=threads)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            vals.append(float(res["final_now_ns"].astype(np.float64).sum()) / 1e9 / dt)
            preds.append(float(res["steps"].sum()) / dt)
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": "emulated virtual-sec/wall-sec over config sweep", "value": round(v, 1),
        "unit": "virtual-s/wall-s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "int64+f64",
        "data": "synthetic", "config": config, "steps_per_s": round(statistics.median(preds), 1),
        "cpu_baseline": {"value": round(v, 1), "unit": "virtual-s/wall-s", "cores": threads, "kind": "port",
                         "sample": f"{sample} configs per step of {n} (C oracle restating oracle.simulate)"},
        "e2e": {"value": round(v, 1), "unit": "virtual-s/wall-s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def init_dist(args, world):
    """One process per GPU under torchrun (also at WORLD_SIZE 1, so a 1-rank NCCL run
    exercises the same collective path); `--share-device` puts every rank on cuda:0 with
    gloo collectives on host tensors (a one-GPU dry run of the multi-rank path)."""
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    on = "WORLD_SIZE" in os.environ
    if not on:
        return False, torch.device("cuda", 0), torch.device("cuda", 0)
    if args.share_device:
        dist.init_process_group("gloo")
        return True, torch.device("cuda", 0), torch.device("cpu")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    return True, dev, dev


def all_reduce(vals, op, cdev):
    import torch
    import torch.distributed as dist

    t = torch.tensor(vals, dtype=torch.float64, device=cdev)
    dist.all_reduce(t, op=op)
    return [float(x) for x in t.cpu().tolist()]


def ksim_profile(sw, device):
    """Per-config cycles and loop iterations of one extra (untimed) launch with
    tw_sim_set_profile: cycles per event-loop iteration, and the heaviest config."""
    import torch

    from paper_2601_00397_b200 import _lib
    from paper_2601_00397_b200.sweep import DeviceSweep

    d = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, device=device, per_request=True)
    prof = torch.zeros(16 * len(sw), dtype=torch.int64, device=device)
    _lib.load().tw_sim_set_profile(prof.data_ptr())
    try:
        d.run()
        torch.cuda.synchronize(device)
    finally:
        _lib.load().tw_sim_set_profile(None)
    pr = prof.view(-1, 16).cpu().numpy()
    cyc, iters = pr[:, 0].astype(np.float64), (pr[:, 1] + pr[:, 2]).astype(np.float64)
    del d
    return cyc, iters


def time_alone(sw, device, reps=3):
    """Mean CUDA-event time of one sweep launched alone (L2 flushed between launches)."""
    import torch

    from paper_2601_00397_b200.sweep import DeviceSweep

    d = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, device=device, per_request=True)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=device)
    durs = time_kernel_steps(d.run, reps, 1, flush, torch.cuda.current_stream(device))
    del d, flush
    return sum(durs) / len(durs)


def issue_roofline(kernel_key, ms, sm_mhz, sms, extra):
    """Issue-slot roofline of the event loop: warp instructions per launch (ncu count of this
    code version, profiles/traffic.json) / live launch time, against 4 schedulers x 1 issue
    per cycle x SMs x the SM clock sampled during the timed region."""
    issue = measured_issue(kernel_key) or {}
    inst = issue.get("inst_executed")
    clock = (sm_mhz or 1965.0) * 1e6
    peak = sms * 4 * clock
    out = {"bound": "issue", "unit": "warp-inst/s", "peak": round(peak, 1),
           "peak_source": f"{sms} SMs x 4 schedulers x 1 warp-inst/cycle x {clock / 1e6:.0f} MHz (sampled)"}
    if inst:
        ach = inst / (ms / 1e3)
        out |= {"achieved": round(ach, 1), "frac": round(ach / peak, 4), "inst_per_launch": int(inst)}
    out |= {k: v for k, v in issue.items() if k not in ("inst_executed",)}
    return out | extra


def ksim_roofline(sw, dev, ms, device, peak_gbs, sm_mhz, key, heavy_alone=True):
    """The dominant kernel's line: the issue-slot roofline it is bound by, its HBM numbers
    (tiny: the loop is not bandwidth-bound), cycles per loop iteration and the critical
    chain (the heaviest config alone vs the whole sweep)."""
    import torch

    from paper_2601_00397_b200 import _lib

    launch = _lib.last_sim_launch()
    n_req = int(dev.req_base[-1])
    alg_bytes = (sw.cfgs.nbytes + 64 * len(sw) + 16 * n_req + 16 * n_req
                 + dev.stage_bytes * (launch["grid"] if launch["variant"] == "latency" else 1))
    ach = alg_bytes / (ms / 1e3) / 1e9
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    cyc, iters = ksim_profile(sw, device)
    heavy = int(np.argmax(cyc))
    chain = {"heaviest_config": heavy, "heaviest_label": sw.configs[heavy].label,
             "heaviest_cycles_in_sweep": int(cyc[heavy]), "sweep_ms": round(ms, 4)}
    if heavy_alone:  # the serial loop (one warp), as the sweep runs it
        with _Env(TWB_SIM_SEG=0):
            chain["heaviest_alone_ms"] = round(time_alone(sw.subset([heavy]), device), 4)
    extra = {
        "kernel": "k_sim", "launch": launch, "traffic": measured_traffic(key),
        "cycles_per_iteration": round(float(cyc.sum() / max(iters.sum(), 1)), 1),
        "iterations_per_config_mean": round(float(iters.mean()), 1),
        "critical_chain": chain,
        "hbm": {"achieved": round(ach, 3), "peak": peak_gbs, "unit": "GB/s", "frac": round(ach / peak_gbs, 6),
                "algorithmic_bytes_per_launch": int(alg_bytes),
                "note": "not the bound: configs are serial event loops whose state stays in registers, "
                        "shared memory and L2"},
    }
    return issue_roofline(key, ms, sm_mhz, sms, extra)


def scaling_projection(full, vsec, device, worlds=(2, 4, 8)):
    """Strong scaling of config 5 projected from this GPU: every LPT shard rank r of N would
    run (the same partition bench.py uses under torchrun), each timed ALONE here. Ranks
    share nothing until the final records gather, so the N-GPU step time is the slowest
    shard (plus the gather, measured at N > 1 in e2e)."""
    from paper_2601_00397_b200.distributed import partition
    from paper_2601_00397_b200.sweep import estimate_cost

    cost = estimate_cost(full.pset, full.cfgs, full.workloads)
    out = {"method": "each LPT shard of N timed alone on this B200 (CUDA events, mean of 3 after 1 warm-up)"}
    for N in worlds:
        shards = partition(cost, N)
        ms = [time_alone(full.subset(s), device) for s in shards]
        c = [float(cost[s].sum()) for s in shards]
        out[f"N{N}"] = {"shard_ms": [round(x, 3) for x in ms], "ms_per_step": round(max(ms), 3),
                        "value": round(vsec / (max(ms) / 1e3), 1),
                        "predicted_cost_imbalance": round(max(c) / (sum(c) / N) - 1, 5),
                        "measured_shard_imbalance": round(max(ms) / (sum(ms) / N) - 1, 4)}
    return out


def measure_sweep(sw, args, world, rank, device, cdev, dist_on, label):
    """The timed step of one sweep: device-resident value (kernel only, CUDA events, L2
    flushed) and e2e through the host API (H2D of inputs, kernel, outputs to pinned host
    memory, and at N > 1 the NCCL all-gather + merge of every rank's records)."""
    import torch

    from paper_2601_00397_b200 import _lib
    from paper_2601_00397_b200.distributed import gather_records_device
    from paper_2601_00397_b200.sweep import DeviceSweep, HostSweep

    MAX, SUM = None, None
    if dist_on:
        import torch.distributed as dist

        MAX, SUM = dist.ReduceOp.MAX, dist.ReduceOp.SUM
    dev = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, device=device, per_request=True)
    stream = torch.cuda.current_stream(device)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=device)

    def barrier():
        if dist_on:
            torch.distributed.barrier()

    barrier()
    torch.cuda.synchronize(device)
    launches0 = _lib.launch_count()
    with ClockSampler(device.index or 0) as clk:
        durs = time_kernel_steps(dev.run, args.steps, args.warmup, flush, stream)
    torch.cuda.synchronize(device)
    barrier()
    launches = _lib.launch_count() - launches0 - args.warmup
    ms = sum(durs) / len(durs)
    out = dev.fetch()
    if not (out.results["status"] == 0).all():
        raise SystemExit(f"rank {rank}: {int((out.results['status'] != 0).sum())} configs of {label} did not finish OK")
    vsec, steps = out.virtual_seconds(sw.cfgs["epoch_ns"]), float(out.predictions)
    ms_max = ms
    max_local = len(sw)
    if dist_on:
        ms_max, = all_reduce([ms], MAX, cdev)
        vsec, steps = all_reduce([vsec, steps], SUM, cdev)
        max_local = int(all_reduce([len(sw)], MAX, cdev)[0])
    res = {"dev": dev, "out": out, "ms": ms, "ms_max": ms_max, "vsec": vsec, "steps": steps, "launches": launches,
           "clocks": clk.summary(), "flush": flush}
    if args.no_e2e:
        res["e2e"] = None
        return res
    host = HostSweep(sw.pset, sw.workloads, sw.cfgs, device=device, per_request=True)
    # the streamed mode keeps its records in pull order (host.perm): ids follow them
    rec_ids = np.asarray(sw.global_ids, np.int64)
    if host.perm is not None:
        rec_ids = rec_ids[host.perm]
    ids_dev = torch.from_numpy(rec_ids).to(cdev)
    merged_host = torch.empty((sw.n_global, 8), dtype=torch.int64, pin_memory=True) if dist_on else None
    e_durs = []
    for i in range(args.warmup + args.steps):
        flush_l2(flush)
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        host.run_from_host()
        if dist_on:  # the sweep's one collective: records of every rank, merged by config id
            recs = host.d_res if cdev.type == "cuda" else host.d_res.cpu()
            merged, _ = gather_records_device(ids_dev, recs, sw.n_global, max_local, cdev)
            merged_host.copy_(merged, non_blocking=True)
        b.record(stream)
        b.synchronize()
        if i >= args.warmup:
            e_durs.append(a.elapsed_time(b))
    e_ms = sum(e_durs) / len(e_durs)
    hr = host.host_results()
    h_first, h_finish = host.host_stamps()
    if not (hr == out.results).all() or not np.array_equal(h_finish, out.finish_ns) or \
            not np.array_equal(h_first, out.first_ns):
        raise SystemExit(f"rank {rank}: e2e host results differ from the device run")
    d2h = host.d2h_bytes
    if dist_on:
        from paper_2601_00397_b200._lib import SIM_RESULT_DTYPE

        m = merged_host.numpy().view(np.uint8).reshape(-1).view(SIM_RESULT_DTYPE)
        if int((m["status"] == 0).sum()) != sw.n_global or int((m["steps"] > 0).sum()) != sw.n_global:
            raise SystemExit(f"rank {rank}: merged records incomplete")
        if not (m[sw.global_ids] == out.results).all():
            raise SystemExit(f"rank {rank}: merged records differ from this rank's")
        e_ms, = all_reduce([e_ms], MAX, cdev)
        d2h += merged_host.numel() * 8
        res["merged"] = m
    res["e2e"] = {"value": round(vsec / (e_ms / 1e3), 1), "unit": "virtual-s/wall-s",
                  "h2d_bytes_per_step": host.h2d_bytes, "d2h_bytes_per_step": int(d2h),
                  "ms_per_step": round(e_ms, 4), "steps_per_s": round(steps / (e_ms / 1e3), 1),
                  "outputs": ("zero-copy: the kernel stores records and stamps into pinned host memory"
                              if host.zero_copy else
                              "streamed: records into pinned host memory, and each finished prefix of configs' stamps "
                              "copied on a second stream while the kernel runs (the last ones after it)")
                  + ("; then the NCCL all-gather of every rank's records and the merge by config id, on device, "
                     "copied to host" if dist_on else "")}
    del host
    return res


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch

    world, rank, local = dist_env()
    dist_on, device, cdev = init_dist(args, world)
    torch.cuda.set_device(device)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "fallback": True}
    peak_gbs = float(peaks["hbm_gbs"])

    sw, config, scaling = build_workload(args, world, rank)
    head = measure_sweep(sw, args, world, rank, device, cdev, dist_on, config["workload"])
    ms_max, vsec, steps_total = head["ms_max"], head["vsec"], head["steps"]
    value = vsec / (ms_max / 1e3)
    key = "k_sim" if args.sweep == "1024" else "k_sim_65536"
    roof = ksim_roofline(sw, head["dev"], head["ms"], device, peak_gbs, head["clocks"].get("sm_mhz"), key,
                         heavy_alone=(rank == 0))

    extra = {}
    solo = rank == 0 and world == 1
    if rank == 0:
        flush = head["flush"]
        stream = torch.cuda.current_stream(device)
        for name, fn in (("predictor_roofline", lambda: predictor_roofline(device, peak_gbs)),
                         ("extraction_roofline", lambda: extraction_roofline(device, peak_gbs)),
                         ("timekeeper_roofline", lambda: timekeeper_roofline(device, peak_gbs)),
                         ("workload_generation", lambda: workload_generation(device)),
                         ("metrics_reduction", lambda: metrics_roofline(head["dev"], args, flush, stream, peak_gbs))):
            try:
                extra[name] = fn()
            except Exception as exc:  # report, never hide
                extra[name] = {"error": repr(exc)}
    if solo and args.sweep == "65536" and not args.no_projection:
        try:
            extra["scaling_projection"] = scaling_projection(sw, vsec, device)
        except Exception as exc:
            extra["scaling_projection"] = {"error": repr(exc)}
    if solo and args.sweep == "65536" and not args.no_config4:
        try:
            extra["config4"] = config4_block(args, device, cdev, peak_gbs)
        except Exception as exc:
            extra["config4"] = {"error": repr(exc)}
    if solo and not args.no_configs13:
        try:
            extra["configs_1_3"] = configs_1_3(device)
        except Exception as exc:
            extra["configs_1_3"] = {"error": repr(exc)}
    cpu = None
    if solo and not args.no_cpu_baseline:
        cpu = cpu_baseline(sw, args.cpu_budget_s, os.cpu_count() or 1)
        try:
            cpu["python"] = cpu_baseline_python(sw, head["out"].results)
        except Exception as exc:
            cpu["python"] = {"error": repr(exc)}

    if rank == 0:
        line = {
            "metric": "emulated virtual-sec/wall-sec over config sweep", "value": round(value, 1),
            "unit": "virtual-s/wall-s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_max, 4), "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "int64+f64", "data": "synthetic", "config": config,
            "steps_per_s": round(steps_total / (ms_max / 1e3), 1), "emulated_steps_per_step": int(steps_total),
            "virtual_s_per_step": round(vsec, 3), "gpu_launches": int(head["launches"]), "clocks": head["clocks"],
            "e2e": head["e2e"], "roofline": roof, "cpu_baseline": cpu, **extra,
        }
        print(json.dumps(line), flush=True)
    if dist_on:
        torch.distributed.destroy_process_group()


class _Env:
    """Library switches for one measurement (read by libtwb200 at launch time)."""

    def __init__(self, **env):
        self.env = {k: str(v) for k, v in env.items()}

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.env}
        os.environ.update(self.env)

    def __exit__(self, *exc):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def seg_stats(sw, device):
    """Busy-period segment statistics of one extra (untimed) launch (tw_sim_set_seg_stats)."""
    import torch

    from paper_2601_00397_b200 import _lib
    from paper_2601_00397_b200.sweep import DeviceSweep

    d = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, device=device, per_request=True)
    st = torch.zeros(8 * len(sw), dtype=torch.int32, device=device)
    _lib.load().tw_sim_set_seg_stats(st.data_ptr())
    try:
        d.run()
        torch.cuda.synchronize(device)
    finally:
        _lib.load().tw_sim_set_seg_stats(None)
    path = _lib.last_sim_launch()["variant"]
    s = st.view(-1, 8).cpu().numpy().astype(np.int64).sum(0)
    del d
    if path != "segments":
        return {"path": path}
    return {"path": path, "segments": int(s[0]), "joined_from_segment_runs": int(s[1]),
            "serial_pieces_in_join": int(s[2]), "timekeeper_carry_refused": int(s[3]),
            "segments_out_of_room": int(s[4]), "stops_not_regeneration_points": int(s[5])}


def seg_roofline(sw, ms, device, sm_mhz, key):
    """The segmented path's line (latency regime): the issue-slot roofline of its four kernels
    together (k_seg_plan, k_sim_seg, k_seg_tk, k_sim_join; ncu instruction count of this code
    version, profiles/traffic.json) over the live launch time, the segment statistics, and
    the serial loop (one warp per config, TWB_SIM_SEG=0) timed beside it with its critical
    chain (the heaviest config alone)."""
    import torch

    from paper_2601_00397_b200 import _lib

    launch = _lib.last_sim_launch()
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    stats = seg_stats(sw, device)
    with _Env(TWB_SIM_SEG=0):
        serial_ms = time_alone(sw, device)
        cyc, iters = ksim_profile(sw, device)
        heavy = int(np.argmax(cyc))
        heavy_serial = time_alone(sw.subset([heavy]), device)
    heavy_seg = time_alone(sw.subset([heavy]), device)
    extra = {"kernel": "k_seg_plan + k_sim_seg + k_seg_tk + k_sim_join", "launch": launch,
             "segments": stats,
             "serial_loop": {"ms": round(serial_ms, 4), "speedup": round(serial_ms / ms, 3),
                             "cycles_per_iteration": round(float(cyc.sum() / max(iters.sum(), 1)), 1),
                             "heaviest_config": heavy, "heaviest_label": sw.configs[heavy].label,
                             "heaviest_alone_ms": round(heavy_serial, 4),
                             "heaviest_alone_segmented_ms": round(heavy_seg, 4)},
             "meaning": "each config's arrivals split into busy-period segments simulated in parallel and "
                        "joined: the sweep is issue-bound instead of bound by its longest serial chain"}
    return issue_roofline(key, ms, sm_mhz, sms, extra)


def config4_block(args, device, cdev, peak_gbs):
    """BASELINE config 4 (the 1,024-config sweep on one B200): the same measurements as
    the headline at N = 1, reported beside it."""
    from paper_2601_00397_b200 import _lib, presets

    sw = presets.sweep_1024(model="8b", seed=1)
    sw.global_ids = np.arange(len(sw), dtype=np.int64)
    sw.n_global = len(sw)
    r = measure_sweep(sw, args, 1, 0, device, cdev, False, "config 4")
    sm_mhz = r["clocks"].get("sm_mhz")
    if _lib.last_sim_launch()["variant"] == "segments":
        roof = seg_roofline(sw, r["ms"], device, sm_mhz, "k_sim_seg")
    else:
        roof = ksim_roofline(sw, r["dev"], r["ms"], device, peak_gbs, sm_mhz, "k_sim")
    return {"workload": "BASELINE config 4: 1,024 configs (Llama-3-8B tables, 1,000 requests, qps 8, seed 1)",
            "value": round(r["vsec"] / (r["ms_max"] / 1e3), 1), "unit": "virtual-s/wall-s",
            "ms_per_step": round(r["ms_max"], 4), "steps_per_s": round(r["steps"] / (r["ms_max"] / 1e3), 1),
            "e2e": r["e2e"], "roofline": roof, "clocks": r["clocks"]}


if __name__ == "__main__":
    main()
