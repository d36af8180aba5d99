"""Busy-period segments of the event loop (latency regime, sim_seg.cu): the speculative
segmented run must equal the serial loop (and the C oracle) record for record and stamp
for stamp, through every path of the join pass: clean boundaries, overruns into the next
segment, boundaries that are not regeneration points of the next run (serial pieces),
segments that run out of log or overrun room, and configs that stop early."""

from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELDS = ("status", "final_now_ns", "steps", "events", "digest", "tk_seq", "tk_offset_ns", "tk_wall_ns",
          "pred_code")


def _run(sw_pset, wl, cfgs, env=None):
    """One DeviceSweep launch under `env` (library switches are read at launch time);
    returns (SweepResult, launches of that tw_sim_many)."""
    from paper_2601_00397_b200 import _lib
    from paper_2601_00397_b200.sweep import DeviceSweep

    env = env or {}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        dev = DeviceSweep(sw_pset, wl, cfgs, per_request=True)
        n0 = _lib.launch_count()
        dev.run()
        n = _lib.launch_count() - n0
        out = dev.fetch()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return out, n


def _same(a, b):
    for f in FIELDS:
        assert np.array_equal(a.results[f], b.results[f]), f
    assert np.array_equal(a.first_ns, b.first_ns)
    assert np.array_equal(a.finish_ns, b.finish_ns)


def _serial_and_segmented(pset, wl, cfgs, **env):
    ser, n_ser = _run(pset, wl, cfgs, {"TWB_SIM_SEG": "0"})
    seg, n_seg = _run(pset, wl, cfgs, {k: str(v) for k, v in env.items()})
    assert n_ser == 1 and n_seg == 4, (n_ser, n_seg)  # plan + segments + Timekeeper replays + join
    _same(seg, ser)
    return seg


def test_segmented_sweep_1024_equals_serial_loop():
    from paper_2601_00397_b200 import presets

    sw = presets.sweep_1024()
    out = _serial_and_segmented(sw.pset, sw.workloads, sw.cfgs)
    assert (out.results["status"] == 0).all()


@pytest.mark.parametrize("name", ["config1", "config2", "config3"])
def test_segmented_single_configs_equal_oracle(name):
    """BASELINE configs 1-3 (one config each: up to 256 segments over its arrivals)."""
    from oracle import oracle as orc
    from paper_2601_00397_b200 import presets

    sw = getattr(presets, name)()
    out, n = _run(sw.pset, sw.workloads, sw.cfgs)
    assert n == 4
    res, _, first, finish = orc.sim_many(sw.pset.blob, sw.cfgs, sw.workloads.wl_off, sw.workloads.offset_ns,
                                         sw.workloads.prompt, sw.workloads.output, per_request=True)
    for f in FIELDS:
        assert np.array_equal(out.results[f], res[f]), f
    k = len(out.first_ns)
    assert np.array_equal(out.first_ns, first[:k]) and np.array_equal(out.finish_ns, finish[:k])


@pytest.mark.parametrize("w,capdiv", [(256, 1), (64, 4), (256, 1000)])
def test_segmented_overruns_and_overflows_equal_serial(w, capdiv):
    """Config 3's heavy load (2.6% of arrivals find the engine empty) with 256 segments:
    about half the boundaries overrun (side-buffer stamps, serial pieces where the next
    run was not empty at the stop); capdiv shrinks every segment's log and overrun room
    (4: some overflow, 1000: all do, so the join pass re-runs from each last
    regeneration point)."""
    from paper_2601_00397_b200 import presets

    sw = presets.config3()
    _serial_and_segmented(sw.pset, sw.workloads, sw.cfgs, TWB_SIM_SEG_W=w, TWB_SIM_SEG_CAPDIV=capdiv)
    sub = presets.sweep_1024().subset(range(0, 1024, 16))
    _serial_and_segmented(sub.pset, sub.workloads, sub.cfgs, TWB_SIM_SEG_W=w, TWB_SIM_SEG_CAPDIV=capdiv)


def test_segmented_configs_that_stop_early_equal_serial():
    """Stalls (a prompt larger than the KV capacity) and prediction errors (a Linear model
    whose duration turns negative for large prefill batches) part-way through the
    arrivals: records equal the serial loop's, and stamps a speculative segment wrote past
    the stop are reset (both runs start from unset stamps)."""
    from paper_2601_00397_b200 import presets
    from paper_2601_00397_b200.predictor import LinearPredictor, PredictorSet

    sw = presets.config1()
    cfgs = np.repeat(sw.cfgs, 6)
    cfgs["kv_capacity_blocks"][0] = 100  # 1,600 tokens: a longer prompt can never be admitted
    cfgs["kv_capacity_blocks"][1] = 126
    cfgs["max_batch_tokens"][2:4] = 4096
    cfgs["chunk_size"][2:4] = 4096
    pset = PredictorSet([sw.pset.predictors[cfgs["pred_id"][0]], LinearPredictor(10000.0, -4.9, 30.0),
                         LinearPredictor(9000.0, -4.0, 20.0)])
    cfgs["pred_id"][:] = 0
    cfgs["pred_id"][2] = 1  # negative once a batch holds > ~2,040 prefill tokens
    cfgs["pred_id"][3] = 2
    cfgs["max_running"][4] = 1  # plain configs next to them
    out = _serial_and_segmented(pset, sw.workloads, cfgs)
    st = out.results["status"]
    assert st[0] != 0 and st[1] != 0 and st[2] != 0 and st[3] != 0 and st[4] == 0 and st[5] == 0, st


def test_segmented_timekeeper_off_and_mixed_workloads_equal_oracle():
    """Configs without the Timekeeper, several workloads of different sizes (including
    empty and one-request workloads) in one launch."""
    from oracle import oracle as orc
    from paper_2601_00397_b200 import presets
    from paper_2601_00397_b200.workload import WorkloadSpec, pack_arrays, poisson_arrays

    docs = [presets.workload_doc(seed=s, n=n) for s, n in ((3, 0), (4, 1), (5, 17), (6, 400), (7, 2500))]
    wl = pack_arrays([poisson_arrays(WorkloadSpec.from_doc(d)) for d in docs])
    base = presets.sweep_1024().subset(range(0, 1024, 64))
    cfgs = np.tile(base.cfgs, len(docs))
    cfgs["workload_id"] = np.repeat(np.arange(len(docs)), len(base.cfgs))
    cfgs["flags"][::2] = 0  # Timekeeper off on every other config
    out, n = _run(base.pset, wl, cfgs)
    assert n == 4
    res, _, first, finish = orc.sim_many(base.pset.blob, cfgs, wl.wl_off, wl.offset_ns, wl.prompt, wl.output,
                                         per_request=True)
    for f in FIELDS:
        assert np.array_equal(out.results[f], res[f]), f
    k = len(out.first_ns)
    assert np.array_equal(out.first_ns, first[:k]) and np.array_equal(out.finish_ns, finish[:k])


def _random_sweep(seed):
    """A random sweep: engine configs (chunk, budget, max_running, KV capacity down to
    stalls, both policies, TP x PP, Timekeeper on/off, cooldown 0 to 2 ms, live epochs, a
    few invalid configs), workloads of 0-600 requests at qps 1-64 with short and long
    prompts, Table / Linear / Constant predictors; plus random segment-path knobs."""
    from paper_2601_00397_b200 import presets
    from paper_2601_00397_b200.predictor import ConstantPredictor, LinearPredictor, PredictorSet
    from paper_2601_00397_b200.sweep import EngineConfig, SchedulingPolicy, SweepConfig, config_array
    from paper_2601_00397_b200.workload import WorkloadSpec, pack_arrays, poisson_arrays

    rng = np.random.default_rng(1000 + seed)
    docs = []
    for w in range(6):
        lo = int(rng.choice([1, 16, 64, 512]))
        docs.append({"source": "poisson", "qps": float(rng.choice([1, 4, 16, 64])), "seed": int(rng.integers(1, 10**6)),
                     "num_requests": int(rng.choice([0, 1, 37, 200, 600])),
                     "prompt_tokens": {"kind": "uniform", "low": lo, "high": lo + int(rng.integers(1, 3000))},
                     "output_tokens": {"kind": "uniform", "low": 1, "high": int(rng.integers(2, 400))}})
    wl = pack_arrays([poisson_arrays(WorkloadSpec.from_doc(d)) for d in docs])
    tables = presets.calibration_set().predictors
    pset = PredictorSet(list(tables) + [LinearPredictor(3000.0, 2.5, 40.0), ConstantPredictor(9000)])
    cfgs = []
    for k in range(192):
        chunk = int(rng.choice([32, 128, 512, 2048]))
        eng = EngineConfig(chunk_size=chunk, max_batch_tokens=chunk * int(rng.choice([1, 2, 8])),
                           max_running=int(rng.choice([1, 4, 32, 256])), kv_block_tokens=int(rng.choice([8, 16])),
                           kv_capacity_blocks=int(rng.choice([300, 4000, 1 << 20])),
                           policy=SchedulingPolicy.MIXED if rng.random() < 0.5 else SchedulingPolicy.PREFILL_PRIORITIZED,
                           workers_per_replica=int(rng.choice([1, 2, 8])), pp_stages=int(rng.choice([1, 2, 3])))
        cfgs.append(SweepConfig(engine=eng, pred_id=int(rng.integers(0, len(pset.predictors))),
                                workload_id=int(rng.integers(0, len(docs))), timekeeper=bool(rng.random() < 0.8),
                                tk_cooldown_ns=int(rng.choice([0, 1, 500_000, 2_000_000])),
                                epoch_ns=int(rng.choice([0, 1_790_000_000_000_000_000]))))
    ca = config_array(cfgs)
    ca["chunk_size"][rng.random(len(ca)) < 0.03] = 0  # a few invalid configs (TW_SIM_BAD_CONFIG)
    env = {"TWB_SIM_SEG_W": int(rng.choice([1, 2, 5, 17, 64])), "TWB_SIM_SEG_CAPDIV": int(rng.choice([1, 1, 3, 1000]))}
    return pset, wl, ca, env


@pytest.mark.parametrize("seed", range(24))
def test_segmented_random_sweeps_equal_serial(seed):
    """Random sweeps (_random_sweep) with random segment counts and room divisors: the
    segmented run equals the serial loop."""
    pset, wl, ca, env = _random_sweep(seed)
    _serial_and_segmented(pset, wl, ca, **env)


@pytest.mark.parametrize("seed", range(24))
def test_random_sweeps_equal_oracle_in_every_loop(seed):
    """The same random sweeps against the C oracle through each event loop: the segments
    (default), the serial latency variant (TWB_SIM_SEG=0) and, with the configs repeated
    past 8 per SM, the throughput variant."""
    import torch

    from oracle import oracle as orc
    from paper_2601_00397_b200 import _lib

    pset, wl, ca, _ = _random_sweep(seed)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    big = np.tile(ca, (8 * sms) // len(ca) + 1)
    for cfgs, env, variant in ((ca, {}, "segments"), (ca, {"TWB_SIM_SEG": "0"}, "latency"), (big, {}, "throughput")):
        out, _ = _run(pset, wl, cfgs, env)
        assert _lib.last_sim_launch()["variant"] == variant
        res, _, first, finish = orc.sim_many(pset.blob, cfgs, wl.wl_off, wl.offset_ns, wl.prompt, wl.output,
                                             per_request=True)
        for f in FIELDS:
            assert np.array_equal(out.results[f], res[f]), (variant, f)
        ok = (res["status"] & 0xFF) == 0
        for c in np.flatnonzero(ok):  # stamps of runs that completed (stopped runs leave theirs unset)
            lo, hi = out.req_base[c], out.req_base[c + 1]
            assert np.array_equal(out.first_ns[lo:hi], first[lo:hi]) and np.array_equal(out.finish_ns[lo:hi], finish[lo:hi]), (variant, c)
