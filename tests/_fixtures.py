"""Loaders for the golden fixtures (tests/golden/*, produced by make_golden.py from
the reference implementation) and builders of the matching engine inputs."""

from __future__ import annotations

import functools
import json
import os

import numpy as np

from paper_2601_00397_b200 import calibration
from paper_2601_00397_b200._lib import SIM_CFG_DTYPE, TK_OP_DTYPE, TW_SIM_TIMEKEEPER
from paper_2601_00397_b200.predictor import (
    ConstantPredictor,
    LinearPredictor,
    PredictorSet,
    TablePredictor,
)
from paper_2601_00397_b200.sweep import EngineConfig, SweepConfig, config_array
from paper_2601_00397_b200.workload import Arrival, WorkloadSpec, generate_arrivals, pack_arrivals

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _npz(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@functools.lru_cache(maxsize=None)
def predictor_golden(name: str = "predictor.npz"):
    """predictor.npz; predictor_neg.npz: tables with negative rows."""
    z = _npz(name)
    specs = json.loads(bytes(z["specs"]).decode())
    preds = [predictor_from_spec(s) for s in specs]
    return specs, preds, z["P"], z["D"], z["C"], z["desc"], z["expected"]


def predictor_from_spec(s):
    if s["kind"] == "constant":
        return ConstantPredictor(s["us"])
    if s["kind"] == "linear":
        return LinearPredictor(*s["coef"])
    if "rows" in s:
        return TablePredictor({(p, d): v for p, d, v in s["rows"]}, allow_extrapolation=s["ext"])
    return TablePredictor.from_csv(calibration.csv_path(*s["table"]), allow_extrapolation=s.get("ext", True))


@functools.lru_cache(maxsize=None)
def barrier_golden(name: str = "barrier.npz"):
    """barrier.npz: 1-5 actors (run_random_schedule); barrier_wide.npz: 6-32 clients;
    barrier_xwide.npz: 33-257 clients, up to 48 groups (tw_tk_replay_wide)."""
    z = _npz(name)
    ops = z["ops"].view(TK_OP_DTYPE)
    return {k: z[k] for k in z.files if k != "ops"} | {"ops": ops}


@functools.lru_cache(maxsize=None)
def resolve_golden():
    """Single resolve rounds at A = 9, 17, 32 computed by the reference BarrierCore._resolve."""
    z = _npz("resolve_wide.npz")
    return {A: {k: z[f"{k}{A}"] for k in ("pending", "elig", "in", "out", "flag")} for A in (9, 17, 32)}


def resolve_xwide_golden():
    """The same at A = 33, 65, 257 with [C, ceil(A/32)] eligibility words (tw_tk_resolve_wide)."""
    z = _npz("resolve_xwide.npz")
    return {A: {k: z[f"{k}{A}"] for k in ("pending", "elig", "in", "out", "flag")} for A in (33, 65, 257)}


@functools.lru_cache(maxsize=None)
def oracle_golden():
    z = _npz("oracle.npz")
    cases = json.loads(bytes(z["cases"]).decode())
    return cases, z["events"], z["ev_off"]


SWEEP_WORKLOAD = {
    "source": "poisson", "qps": 8, "seed": 1, "num_requests": 1000,
    "prompt_tokens": {"kind": "uniform", "low": 64, "high": 2048},
    "output_tokens": {"kind": "uniform", "low": 16, "high": 256},
}


@functools.lru_cache(maxsize=None)
def workload_for(n: int, first: tuple):
    """Regenerate a full-size golden workload (pinned by arrivals.json)."""
    cands = [dict(SWEEP_WORKLOAD), dict(SWEEP_WORKLOAD, qps=4, num_requests=10000)]
    for doc in cands:
        if doc["num_requests"] != n:
            continue
        arr = generate_arrivals(WorkloadSpec.from_doc(doc))
        if (arr[0].offset_ns, arr[0].prompt_tokens, arr[0].output_tokens) == tuple(first):
            return arr
    raise KeyError((n, first))


def case_inputs(case, timekeeper=False):
    """(PredictorSet, PackedWorkloads, cfg array[1]) for one oracle.npz case."""
    if case["arrivals"] is not None:
        arr = [Arrival(r, o, p, q) for r, o, p, q in case["arrivals"]]
    else:
        arr = workload_for(case["workload"]["n"], tuple(case["workload"]["first"]))
    eng = EngineConfig.from_doc(case["engine"])
    pset = PredictorSet([predictor_from_spec(case["pred"])])
    wl = pack_arrivals([arr])
    cfgs = config_array([SweepConfig(engine=eng, epoch_ns=case["epoch"], timekeeper=timekeeper)])
    return pset, wl, cfgs


def case_events(case, events, ev_off):
    i = case["ev_index"]
    return events[ev_off[i] : ev_off[i + 1]]


@functools.lru_cache(maxsize=None)
def tkgrid_golden():
    with open(os.path.join(GOLDEN, "tkgrid.json")) as fh:
        return json.load(fh)


def tk_case_inputs(case):
    doc = {"source": "poisson", "qps": 20, "seed": 5, "num_requests": 120,
           "prompt_tokens": {"kind": "uniform", "low": 16, "high": 900},
           "output_tokens": {"kind": "uniform", "low": 1, "high": 60}} if case["seed"] == 5 else SWEEP_WORKLOAD
    arr = generate_arrivals(WorkloadSpec.from_doc(doc))
    eng = EngineConfig(chunk_size=512, max_batch_tokens=2048, max_running=256, kv_block_tokens=16,
                       kv_capacity_blocks=32768, workers_per_replica=case["tp"], pp_stages=case["pp"])
    ttp, tpp = case.get("table_tp", case["tp"]), case.get("table_pp", case["pp"])
    pset = PredictorSet([TablePredictor.from_csv(calibration.csv_path(case["model"], ttp, tpp),
                                                 allow_extrapolation=True)])
    cfgs = config_array([SweepConfig(engine=eng, epoch_ns=case["epoch"], timekeeper=True,
                                     tk_cooldown_ns=case["cooldown"])])
    return pset, pack_arrivals([arr]), cfgs


@functools.lru_cache(maxsize=None)
def metrics_golden():
    """[(record, oracle case)]: the reference's RunReport.summary() per oracle case."""
    with open(os.path.join(GOLDEN, "metrics.json")) as fh:
        recs = json.load(fh)
    cases = {c["name"]: c for c in oracle_golden()[0]}
    return [(r, cases[r["name"]]) for r in recs]


def caller_order(case, perm):
    """Workloads packed with the golden record's arrival-list order (perm: position ->
    original index, None = the original list), so caller_index orders the TPOT sum."""
    if case["arrivals"] is not None:
        arr = [Arrival(r, o, p, q) for r, o, p, q in case["arrivals"]]
    else:
        arr = workload_for(case["workload"]["n"], tuple(case["workload"]["first"]))
    if perm is not None:
        arr = [arr[i] for i in perm]
    return arr


def assert_summary_equal(rec, golden, what=""):
    """Bit-exact comparison of one RUN_METRICS_DTYPE record with a golden summary."""
    assert int(rec["status"]) == 0, (what, int(rec["status"]))
    for k in ("num_requests", "virtual_elapsed_ns", "output_tokens"):
        assert int(rec[k]) == golden[k], (what, k, int(rec[k]), golden[k])
    assert float(rec["tokens_per_virtual_s"]).hex() == golden["tokens_per_virtual_s"], what
    for m, key in (("ttft", "ttft_ns"), ("e2e", "e2e_ns"), ("tpot", "tpot_ns")):
        if key not in golden:
            assert int(rec[m]["count"]) == 0, (what, m)
            continue
        g = golden[key]
        assert int(rec[m]["count"]) == g["count"], (what, m)
        for f in ("p50", "p90", "p99", "mean"):
            assert float(rec[m][f]).hex() == g[f], (what, m, f, float(rec[m][f]).hex(), g[f])
