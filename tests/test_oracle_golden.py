"""Pin the CPU oracle (oracle/twb_oracle.c) against the reference's own outputs.

The golden vectors come from running the reference implementation
(tests/golden/make_golden.py): predictor.py predict(), BarrierCore under a
FakeClock (pkg/tests/_support.py run_random_schedule seeds 0-1099 + scenarios
after pkg/tests/test_barrier_core.py), oracle.simulate (pkg/tests/test_oracle.py
timelines, the scheduler-agreement workload of pkg/tests/test_engine.py:271-285,
randomized cases, BASELINE configs 1-3 and 1,024-grid samples).
"""

import hashlib
import json
import os

import numpy as np
import pytest

from _fixtures import (
    GOLDEN,
    barrier_golden,
    resolve_golden,
    case_events,
    case_inputs,
    oracle_golden,
    predictor_golden,
    resolve_xwide_golden,
    tk_case_inputs,
    tkgrid_golden,
)
from oracle import oracle as orc
from paper_2601_00397_b200.predictor import PredictorSet
from paper_2601_00397_b200.workload import WorkloadSpec, pack_arrivals, poisson_arrays

STATUS_OF = {0: 0, 1: 1, 2: 2, 3: 3}


def test_oracle_predictor_matches_reference():
    specs, preds, P, D, C, desc, expected = predictor_golden()
    blob = PredictorSet(preds).blob
    got = orc.predict_many(blob, P, D, C, desc)
    bad = np.nonzero(got != expected)[0]
    assert bad.size == 0, [(specs[desc[i]]["name"], P[i], D[i], C[i], got[i], expected[i]) for i in bad[:5]]


def test_oracle_predictor_negative_rows_match_reference():
    """TablePredictor(rows) with negative values (the reference accepts them outside
    from_csv): negative multiples of 1000 ns, a -1 us row that is not a hole."""
    specs, preds, P, D, C, desc, expected = predictor_golden("predictor_neg.npz")
    got = orc.predict_many(PredictorSet(preds).blob, P, D, C, desc)
    assert np.array_equal(got, expected)
    assert ((expected < 0) & (expected % 1000 == 0)).any()


def test_oracle_predictor_empty_batch_code():
    specs, preds, *_ = predictor_golden()
    blob = PredictorSet(preds).blob
    out = orc.predict_many(blob, [0, 0], [0, 0], [-1, -1], [0, len(preds) - 1])
    assert out.tolist() == [-1, -1]


@pytest.mark.parametrize("name", ["barrier.npz", "barrier_wide.npz", "barrier_xwide.npz"])
def test_oracle_barrier_replay_matches_reference(name):
    g = barrier_golden(name)
    ack, events, fin = orc.tk_replay(g["ops"], g["op_off"], g["wall0"], g["cooldown"], g["suppress"])
    assert np.array_equal(ack, g["acks"])
    n = len(g["op_off"]) - 1
    for s in range(n):
        want = g["events"][g["ev_off"][s] : g["ev_off"][s + 1]]
        got = events[s]
        assert len(got) == len(want), s
        got4 = np.stack([got["kind"], got["offset_ns"], got["seq"], got["wall_ns"]], axis=1) if len(got) else np.zeros((0, 4))
        assert np.array_equal(got4, want), s
    assert np.array_equal(np.stack([fin["offset_ns"], fin["seq"], fin["wall_ns"]], axis=1), g["final"])


@pytest.mark.parametrize("A", [9, 17, 32])
def test_oracle_resolve_rounds_match_reference_resolve(A):
    g = resolve_golden()[A]
    st = [g["pending"].copy()] + [g["in"][:, k].copy() for k in range(4)]
    flag = orc.tk_resolve(st[0], g["elig"], A, 500_000, st[1], st[2], st[3], st[4])
    assert np.array_equal(flag, g["flag"])
    assert np.array_equal(np.stack(st[1:], axis=1), g["out"])
    assert (st[0][np.repeat(g["flag"] >= 0, A)] == np.iinfo(np.int64).max).all()


def _check_case(case, res, first, finish, events, ev_all, ev_off):
    st = int(res["status"]) & 0xFF
    assert st == STATUS_OF[case["status"]], (case["name"], st)
    if case["status"] != 0:
        return
    assert int(res["events"]) == case["n_events"], case["name"]
    assert int(np.uint64(res["digest"])) == int(case["digest"]), case["name"]
    assert int(res["final_now_ns"]) == case["final_ts"], case["name"]
    assert int(res["steps"]) == case["steps"], case["name"]
    assert hashlib.sha256(first.astype(np.int64).tobytes()).hexdigest() == case["first_sha"], case["name"]
    assert hashlib.sha256(finish.astype(np.int64).tobytes()).hexdigest() == case["finish_sha"], case["name"]
    if events is not None and "ev_index" in case:
        want = case_events(case, ev_all, ev_off)
        rk = events["req_kind"].astype(np.int64)
        got = np.stack([rk >> 2, rk & 3, events["ts_ns"], events["step"]], axis=1)
        assert np.array_equal(got, want), case["name"]


def test_oracle_simulate_small_cases_event_for_event():
    cases, ev_all, ev_off = oracle_golden()
    small = [c for c in cases if c["arrivals"] is not None]
    assert len(small) >= 80
    for case in small:
        pset, wl, cfgs = case_inputs(case)
        ts, pr, out = wl.workload(0)
        res, first, finish, events = orc.simulate_one(pset.blob, cfgs[0], ts, pr, out, want_events=True)
        _check_case(case, res, first, finish, events, ev_all, ev_off)


@pytest.mark.slow
def test_oracle_simulate_full_size_cases():
    cases, ev_all, ev_off = oracle_golden()
    big = [c for c in cases if c["arrivals"] is None]
    assert len(big) >= 19
    for case in big:
        pset, wl, cfgs = case_inputs(case)
        ts, pr, out = wl.workload(0)
        res, first, finish, _ = orc.simulate_one(pset.blob, cfgs[0], ts, pr, out, want_events=False)
        _check_case(case, res, first, finish, None, ev_all, ev_off)


@pytest.mark.parametrize("case", tkgrid_golden(), ids=lambda c: c["name"])
def test_oracle_timekeeper_grid_matches_reference_barriercore(case):
    pset, wl, cfgs = tk_case_inputs(case)
    ts, pr, out = wl.workload(0)
    res, *_ = orc.simulate_one(pset.blob, cfgs[0], ts, pr, out, want_events=False)
    assert int(res["status"]) == 0
    assert int(np.uint64(res["digest"])) == int(case["digest"])
    assert (int(res["tk_seq"]), int(res["tk_offset_ns"]), int(res["tk_wall_ns"])) == (
        case["seq"], case["offset"], case["wall"]
    )


def test_workload_generator_matches_reference_arrivals():
    with open(os.path.join(GOLDEN, "arrivals.json")) as fh:
        shas = json.load(fh)
    z = np.load(os.path.join(GOLDEN, "arrivals.npz"))
    for name, rec in shas.items():
        if rec["doc"]["num_requests"] > 2000:
            continue  # the 10k-request trace is checked in the slow test
        ts, pr, op = poisson_arrays(WorkloadSpec.from_doc(rec["doc"]))
        assert hashlib.sha256(ts.tobytes() + pr.tobytes() + op.tobytes()).hexdigest() == rec["sha"], name
        if name + "_ts" in z.files:
            assert np.array_equal(ts, z[name + "_ts"])


def test_sim_many_threads_equal_single():
    cases, *_ = oracle_golden()
    small = [c for c in cases if c["arrivals"] is not None][:40]
    from paper_2601_00397_b200.predictor import PredictorSet as PS
    from paper_2601_00397_b200.workload import pack_arrays
    from paper_2601_00397_b200._lib import SIM_CFG_DTYPE

    preds, arrays, cfgs = [], [], np.zeros(len(small), SIM_CFG_DTYPE)
    singles = []
    for i, case in enumerate(small):
        pset, wl, c = case_inputs(case)
        preds.append(pset.predictors[0])
        arrays.append(wl.workload(0))
        cfgs[i] = c[0]
        cfgs[i]["pred_id"] = i
        cfgs[i]["workload_id"] = i
        ts, pr, out = wl.workload(0)
        singles.append(orc.simulate_one(pset.blob, c[0], ts, pr, out, want_events=False)[0])
    blob = PS(preds).blob
    wl = pack_arrays(arrays)
    res, *_ = orc.sim_many(blob, cfgs, wl.wl_off, wl.offset_ns, wl.prompt, wl.output, n_threads=4)
    for i, s in enumerate(singles):
        assert res[i].tobytes() == s.tobytes()


def _oracle_metrics_case(rec, case):
    from _fixtures import caller_order

    pset, wl, cfgs = case_inputs(case)
    ts, pr, out = wl.workload(0)
    res, first, finish, _ = orc.simulate_one(pset.blob, cfgs[0], ts, pr, out, want_events=False)
    arr = caller_order(case, rec["perm"])
    cw = pack_arrivals([arr])  # the engine's sorted order + each request's caller position
    pos = cw.caller_index
    n = len(arr)
    # arrays in the caller's order: engine request e sits at caller position pos[e]
    c_ts, c_out, c_first, c_fin = (np.empty(n, np.int64), np.empty(n, np.int32), np.empty(n, np.int64),
                                   np.empty(n, np.int64))
    c_ts[pos], c_out[pos], c_first[pos], c_fin[pos] = cw.offset_ns, cw.output, first, finish
    return orc.metrics(c_ts, c_out, c_first, c_fin, case["epoch"])


def test_oracle_metrics_match_reference_summaries():
    """orc_metrics == collect_metrics(...).summary() bit for bit (metrics.py:38-253),
    including shuffled arrival lists (ordered TPOT sum); full-size cases: config 1 only."""
    from _fixtures import assert_summary_equal, metrics_golden

    done = 0
    for rec, case in metrics_golden():
        if case["arrivals"] is None and case["name"] != "config1_8b_tp1":
            continue
        assert_summary_equal(_oracle_metrics_case(rec, case), rec["summary"], rec["name"])
        done += 1
    assert done >= 100


@pytest.mark.slow
def test_oracle_metrics_full_size_cases():
    from _fixtures import assert_summary_equal, metrics_golden

    for rec, case in metrics_golden():
        if case["arrivals"] is None:
            assert_summary_equal(_oracle_metrics_case(rec, case), rec["summary"], rec["name"])


def test_oracle_linear_quantisation_extremes():
    """int(round(us)) * 1000 at the edges (predictor.py:137-146): NaN -> ValueError code,
    +-inf -> OverflowError code, finite beyond int64 ns -> engine-limit overflow code,
    -0.5 rounds to 0 (half-even), below that NegativeDuration."""
    from paper_2601_00397_b200.predictor import LinearPredictor

    cases = [(float("nan"), -5), (float("inf"), -6), (float("-inf"), -6), (1e16, -6), (9.3e15, -6),
             (9.2e15, 9_200_000_000_000_000_000), (-0.5, 0), (-0.51, -2), (-1e300, -2), (2.5, 2000), (3.5, 4000)]
    preds = [LinearPredictor(b) for b, _ in cases]
    blob = PredictorSet(preds).blob
    n = len(cases)
    got = orc.predict_many(blob, np.zeros(n, np.int32), np.ones(n, np.int32), np.zeros(n, np.int64),
                           np.arange(n, dtype=np.int32))
    assert got.tolist() == [w for _, w in cases]



@pytest.mark.parametrize("A", [33, 65, 257])
def test_oracle_wide_resolve_rounds_match_reference_resolve(A):
    g = resolve_xwide_golden()[A]
    st = [g["pending"].copy()] + [g["in"][:, k].copy() for k in range(4)]
    flag = orc.tk_resolve_wide(st[0], g["elig"], A, 500_000, *st[1:])
    assert np.array_equal(flag, g["flag"])
    assert np.array_equal(np.stack(st[1:], axis=1), g["out"])
