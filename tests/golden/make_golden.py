"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference read-only from /root/reference/pkg/src (and its test
helpers from /root/reference/pkg/tests/_support.py), runs its predictor,
BarrierCore and oracle.simulate, and writes compact .npz fixtures next to this
file. The GPU box never reads /root/reference: tests only read these fixtures.

Fixtures:
  predictor.npz  queries -> reference predict() ns / exception, per predictor case
  predictor_neg.npz  the same for tables with negative rows (TablePredictor(rows))
  barrier.npz    BarrierCore op streams (run_random_schedule seeds 0-999, the
                 scripted replay harness, hand-written scenarios) -> acks,
                 broadcast/release events, final state
  oracle.npz     oracle.simulate cases -> full event streams (small cases) and
                 digests / spans / per-request stamps (all cases)
  tkgrid.npz     the event loop's Timekeeper actor grid driven through the real
                 BarrierCore on a FakeClock -> (seq, offset, wall) + broadcast digest
  arrivals.npz   generate_arrivals outputs for the sweep workloads
  metrics.json   collect_metrics(...).summary() of the oracle cases (floats as hex),
                 including arrival lists in shuffled order (the TPOT sum is ordered)
  core_log.json.gz full BarrierCore transcripts (every message and ack with all fields,
                 every structured log record, every emitted broadcast/release) of the
                 scripted scenarios and 190 random schedules: pins NativeBarrierCore
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import random
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))
sys.path.insert(0, ROOT)

from timewarp import oracle as ref_oracle  # noqa: E402
from timewarp import predictor as ref_pred  # noqa: E402
from timewarp.engine import EngineConfig, SchedulingPolicy  # noqa: E402
from timewarp.timekeeper import BarrierCore  # noqa: E402
from timewarp.wire import Message, MessageType  # noqa: E402
from timewarp.workload import Arrival, WorkloadSpec, generate_arrivals  # noqa: E402

import _support  # noqa: E402

from oracle.oracle import digest_of_docs, event_hash, M64  # noqa: E402
from paper_2601_00397_b200 import calibration  # noqa: E402
from paper_2601_00397_b200._lib import TK_OP_DTYPE  # noqa: E402

ERR_CODE = {
    "EmptyBatch": -1,
    "NegativeDuration": -2,
    "TableMiss": -3,
}

# ------------------------------------------------------------------------------
# predictor
# ------------------------------------------------------------------------------


class Feat:
    """Duck-typed batch exposing exactly what predict() reads (predictor.py:209-242)."""

    __slots__ = ("total_prefill_tokens", "num_decodes", "total_context")

    def __init__(self, p, d, c):
        self.total_prefill_tokens = p
        self.num_decodes = d
        self.total_context = c

    def is_empty(self):
        return False


def ref_predict(pred, p, d, c) -> int:
    try:
        return pred.predict(Feat(p, d, c))
    except ref_pred.PredictorError as exc:
        return ERR_CODE[type(exc).__name__]


def predictor_cases(rng: np.random.Generator):
    cases = []  # (spec dict, reference predictor)
    test_table = {(0, 1): 100, (0, 8): 800, (512, 1): 2000, (512, 8): 3000, (1024, 1): 4000, (1024, 8): 5200}
    hole = {(0, 1): 100, (512, 1): 2000, (512, 8): 3000}
    for rows, name in ((test_table, "test_table"), (hole, "hole_table")):
        for ext in (False, True):
            cases.append(({"kind": "table", "rows": rows, "ext": ext, "name": f"{name}_ext{int(ext)}"},
                          ref_pred.TablePredictor(rows, allow_extrapolation=ext)))
    for m in calibration.MODELS:
        for tp, pp in calibration.TP_PP_GRID:
            path = calibration.csv_path(m, tp, pp)
            p = ref_pred.TablePredictor.from_csv(path, allow_extrapolation=True)
            cases.append(({"kind": "table", "rows": dict(p._rows), "ext": True,
                           "name": os.path.basename(path)}, p))
    for k in range(4):  # random holey tables
        pax = sorted(set(int(x) for x in rng.integers(0, 5000, size=int(rng.integers(2, 14)))))
        dax = sorted(set(int(x) for x in rng.integers(0, 300, size=int(rng.integers(2, 14)))))
        rows = {}
        for p in pax:
            for d in dax:
                if rng.random() < 0.7:
                    rows[(p, d)] = int(rng.integers(0, 200_000))
        if not rows:
            rows[(pax[0], dax[0])] = 7
        ext = bool(k % 2)
        cases.append(({"kind": "table", "rows": rows, "ext": ext, "name": f"random_holey_{k}"},
                      ref_pred.TablePredictor(rows, allow_extrapolation=ext)))
    lin = [(500.0, 10.0, 150.0, 0.5), (0.0, 0.3, 0.0, 0.0), (-100.0, 0.0, 0.0, 0.0)]
    for _ in range(5):
        lin.append(tuple(float(x) for x in rng.normal(0, 1, 4) * np.array([800, 3, 40, 0.01])))
    lin.append((817.25, 1.0 / 3.0, 37.1, 0.0013))
    for i, co in enumerate(lin):
        cases.append(({"kind": "linear", "coef": co, "name": f"linear_{i}"}, ref_pred.LinearPredictor(*co)))
    for us in (0, 1, 20000):
        cases.append(({"kind": "constant", "us": us, "name": f"constant_{us}"}, ref_pred.ConstantPredictor(us)))
    return cases


def make_predictor_golden(rng):
    cases = predictor_cases(rng)
    specs, P, D, C, I, E = [], [], [], [], [], []
    for ci, (spec, pred) in enumerate(cases):
        specs.append({**spec, "rows": [[k[0], k[1], v] for k, v in spec["rows"].items()]} if "rows" in spec else spec)
        n = 4000 if spec["kind"] == "table" else 3000
        if spec["kind"] == "table":
            ps = sorted({k[0] for k in spec["rows"]})
            ds = sorted({k[1] for k in spec["rows"]})
            qp = rng.integers(0, ps[-1] + 200, size=n)
            qd = rng.integers(0, ds[-1] + 20, size=n)
            # a quarter of the queries sit exactly on axis values (exact hits / edges)
            k = n // 4
            qp[:k] = rng.choice(ps, size=k)
            qd[k : 2 * k] = rng.choice(ds, size=k)
        else:
            qp = rng.integers(0, 8193, size=n)
            qd = rng.integers(0, 513, size=n)
        qc = rng.integers(0, 600_000, size=n)
        for p, d, c in zip(qp.tolist(), qd.tolist(), qc.tolist()):
            P.append(p)
            D.append(d)
            C.append(c)
            I.append(ci)
            E.append(ref_predict(pred, p, d, c))
    np.savez_compressed(
        os.path.join(HERE, "predictor.npz"),
        specs=np.frombuffer(json.dumps(specs).encode(), np.uint8),
        P=np.asarray(P, np.int32), D=np.asarray(D, np.int32), C=np.asarray(C, np.int64),
        desc=np.asarray(I, np.int32), expected=np.asarray(E, np.int64),
    )
    print("predictor:", len(cases), "cases,", len(P), "queries,", sum(e < 0 for e in E), "error codes")


def make_predictor_neg_golden():
    """predictor_neg.npz: TablePredictor(rows) with NEGATIVE values, which the reference
    accepts (it only rejects them in from_csv, predictor.py:164-192): predictions are then
    negative multiples of 1000 ns. Includes a -1 us row (the round-1 device hole marker),
    holes, exact hits, interpolation and nearest-row extrapolation. Same layout as
    predictor.npz; its own seed, so predictor.npz is unchanged."""
    rng = np.random.default_rng(397_2)
    cases = []
    mixed = {(0, 1): -100, (0, 8): 800, (512, 1): -2000, (512, 8): 3000, (1024, 1): -1, (1024, 8): -5200}
    holey = {(0, 1): -1, (512, 1): -2000, (512, 8): 3000, (2048, 4): -7}
    for rows, name in ((mixed, "neg_mixed"), (holey, "neg_holey")):
        for ext in (False, True):
            cases.append(({"kind": "table", "rows": rows, "ext": ext, "name": f"{name}_ext{int(ext)}"},
                          ref_pred.TablePredictor(rows, allow_extrapolation=ext)))
    for k in range(4):
        pax = sorted(set(int(x) for x in rng.integers(0, 5000, size=int(rng.integers(2, 12)))))
        dax = sorted(set(int(x) for x in rng.integers(0, 300, size=int(rng.integers(2, 12)))))
        lo, hi = (-200_000, 200_000) if k % 2 else (-300_000, 0)
        rows = {(p, d): int(rng.integers(lo, hi)) for p in pax for d in dax if rng.random() < 0.75}
        if not rows:
            rows[(pax[0], dax[0])] = -3
        ext = bool(k // 2)
        cases.append(({"kind": "table", "rows": rows, "ext": ext, "name": f"neg_random_{k}"},
                      ref_pred.TablePredictor(rows, allow_extrapolation=ext)))
    specs, P, D, C, I, E = [], [], [], [], [], []
    for ci, (spec, pred) in enumerate(cases):
        specs.append({**spec, "rows": [[k[0], k[1], v] for k, v in spec["rows"].items()]})
        ps = sorted({k[0] for k in spec["rows"]})
        ds = sorted({k[1] for k in spec["rows"]})
        n = 3000
        qp = rng.integers(0, ps[-1] + 200, size=n)
        qd = rng.integers(0, ds[-1] + 20, size=n)
        k = n // 4
        qp[:k] = rng.choice(ps, size=k)
        qd[k : 2 * k] = rng.choice(ds, size=k)
        qc = rng.integers(0, 600_000, size=n)
        for p, d, c in zip(qp.tolist(), qd.tolist(), qc.tolist()):
            P.append(p)
            D.append(d)
            C.append(c)
            I.append(ci)
            E.append(ref_predict(pred, p, d, c))
    np.savez_compressed(
        os.path.join(HERE, "predictor_neg.npz"),
        specs=np.frombuffer(json.dumps(specs).encode(), np.uint8),
        P=np.asarray(P, np.int32), D=np.asarray(D, np.int32), C=np.asarray(C, np.int64),
        desc=np.asarray(I, np.int32), expected=np.asarray(E, np.int64),
    )
    neg = sum(1 for e in E if e < 0 and e % 1000 == 0)
    print("predictor_neg:", len(cases), "cases,", len(P), "queries,", neg, "negative durations,",
          sum(1 for e in E if e < 0 and e % 1000), "error codes")



# ------------------------------------------------------------------------------
# BarrierCore
# ------------------------------------------------------------------------------

ACK = {None: 0, "RegistrationSealed": 1, "NoActors": 2, "UnknownClient": 3, "InvalidState": 4,
       "RoleViolation": 5, "InvalidDelta": 6, "ExpectedMismatch": 7}


class Recorder:
    """Wraps a CoreHarness: records every op as a tw_tk_op plus the ack code."""

    def __init__(self, h):
        self.h = h
        self.ops = []
        self.acks = []
        self.groups = {}
        self.ids = {}  # client id -> registration index, as the core issued them
        orig = h.core.handle

        def handle(msg, reply=None):
            ack = orig(msg, reply)
            self._record(msg, ack)
            return ack

        h.core.handle = handle
        orig_adv = h.clock.advance

        def advance(ns):
            orig_adv(ns)
            self.ops.append((int(ns), 6, 0, 0))
            self.acks.append(0)

        h.clock.advance = advance

    def _cid(self, client_id):
        """Registration index of an id the core issued; -1 for anything else (the core
        answers UnknownClient, e.g. 'actor46' when registration 46 was an observer)."""
        return self.ids.get(client_id or "", -1)

    def _record(self, msg, ack):
        t = msg.type
        err = None if ack.error is None else ack.error.split(":")[0]
        if t is MessageType.REGISTER:
            op = (0, 0 if msg.role == "ACTOR" else 1, 0, 0)
            if err is None:
                self.ids[ack.client_id] = len(self.ids)
        elif t is MessageType.SEAL:
            op = (0, 2, 0, 0)
        elif t is MessageType.JUMP_REQUEST:
            c = self._cid(msg.client_id)
            op = (int(msg.target if msg.target is not None else 0), 3 if c >= 0 else 7, max(c, 0), 0)
        elif t is MessageType.COLLECTIVE_ENTER:
            c = self._cid(msg.client_id)
            g = self.groups.setdefault(msg.group_id, len(self.groups))
            op = (int(msg.expected), 4 if c >= 0 else 7, max(c, 0), g)
        elif t is MessageType.DEREGISTER:
            c = self._cid(msg.client_id)
            op = (0, 5 if c >= 0 else 7, max(c, 0), 0)
        else:
            raise AssertionError(t)
        self.ops.append(op)
        self.acks.append(ACK[err])


def harness_events(h):
    """Broadcast (incl. suppressed) and release records in emission order."""
    out = []
    for r in h.records:
        if r["event"] == "broadcast":
            out.append((0, int(r["offset_ns"]), int(r["seq"]), int(r["wall_ns"])))
        elif r["event"] == "collective_release":
            out.append((1, 0, int(r["generation"]), int(r["wall_ns"])))  # group filled below
    return out


def release_groups(rec, h):
    gids = [rec.groups[r["group_id"]] for r in h.records if r["event"] == "collective_release"]
    return gids


def scenario_streams():
    """Hand-written scenarios after pkg/tests/test_barrier_core.py (with clock advances)."""
    MS, US, WALL0 = 1_000_000, 1_000, 1_000_000_000
    out = []

    def mk(cooldown=500_000, suppress=False):
        h = _support.CoreHarness.build(cooldown_ns=cooldown, suppress=suppress)
        return h, Recorder(h)

    h, r = mk(); a = h.register_actor(); h.seal(); h.jump(a, WALL0 + 40 * MS); out.append((h, r))
    h, r = mk(); a = h.register_actor(); b = h.register_actor(); h.seal(); h.jump(a, WALL0 + 10 * MS); h.jump(b, WALL0 + 20 * MS); out.append((h, r))
    h, r = mk(500 * US); a = h.register_actor(); b = h.register_actor(); h.seal()
    h.jump(a, WALL0 + 100 * MS); h.clock.advance(20 * MS); h.jump(b, WALL0 + 50 * MS); h.jump(a, WALL0 + 100 * MS); h.jump(b, WALL0 + 200 * MS); out.append((h, r))
    h, r = mk(); a = h.register_actor(); h.seal(); h.clock.advance(50 * MS); h.jump(a, WALL0 + 10 * MS); out.append((h, r))
    h, r = mk(500 * US); a = h.register_actor(); h.seal(); h.jump(a, WALL0 + 100 * US); h.jump(a, WALL0 + 300 * US); out.append((h, r))
    h, r = mk(); a = h.register_actor(); b = h.register_actor(); h.seal(); h.jump(a, WALL0 + 10 * MS); h.jump(a, WALL0 + 25 * MS); h.jump(b, WALL0 + 30 * MS); out.append((h, r))
    # roles, sealing, errors
    h, r = mk(); a = h.register_actor(); o = h.register_observer(); h.seal(); h.jump(o, WALL0 + 5 * MS)
    h.core.handle(Message(type=MessageType.REGISTER, role="ACTOR")); h.jump(a, 0); h.jump(a, -5)
    h.core.handle(Message(type=MessageType.JUMP_REQUEST, client_id="actor99", target=5)); h.jump(a, WALL0 + 7 * MS); out.append((h, r))
    h, r = mk(); h.register_observer(); h.seal(); out.append((h, r))
    # deregister unblocks, collectives with exemption and mismatch
    h, r = mk(); a = h.register_actor(); b = h.register_actor(); c = h.register_actor(); h.seal()
    h.jump(a, WALL0 + 10 * MS); h.jump(b, WALL0 + 12 * MS); h.deregister(c); h.deregister(c); h.jump(c, WALL0 + 5 * MS); out.append((h, r))
    h, r = mk(); a = h.register_actor(); b = h.register_actor(); c = h.register_actor(); h.seal()
    h.enter(a, "g", 2); h.jump(b, WALL0 + 3 * MS); h.jump(c, WALL0 + 4 * MS); h.enter(b, "g", 3); h.enter(b, "g", 2)
    h.jump(a, WALL0 + 9 * MS); h.jump(b, WALL0 + 9 * MS); h.enter(c, "g", 1); h.jump(b, WALL0 + 11 * MS); h.jump(a, WALL0 + 12 * MS); h.enter(a, "h", 0); out.append((h, r))
    # suppressed broadcasts
    h, r = mk(500 * US, suppress=True); a = h.register_actor(); h.seal(); h.jump(a, WALL0 + 10 * MS); h.jump(a, WALL0 + 20 * MS); out.append((h, r))
    # zero cooldown, long schedules
    h, r = mk(0); a = h.register_actor(); b = h.register_actor(); h.seal()
    for i in range(1, 40):
        h.jump(a, WALL0 + i * 7 * MS); h.jump(b, WALL0 + i * 5 * MS); h.clock.advance(123_457)
    out.append((h, r))
    return out


def scripted():
    MS, WALL0 = 1_000_000, 1_000_000_000
    h = _support.CoreHarness.build()
    r = Recorder(h)
    a = h.register_actor(); b = h.register_actor(); h.seal()
    h.jump(a, WALL0 + 10 * MS); h.jump(b, WALL0 + 12 * MS); h.jump(a, WALL0 + 30 * MS); h.jump(b, WALL0 + 25 * MS)
    h.enter(a, "g", expected=2); h.enter(b, "g", expected=2)
    h.jump(a, WALL0 + 50 * MS); h.jump(b, WALL0 + 50 * MS); h.deregister(a); h.deregister(b)
    return h, r


def save_streams(streams, name):
    """Pack recorded (harness, recorder, cooldown, suppress) streams into a barrier-format npz."""
    ops, op_off, acks, ev, ev_off, fin, wall0, cool, sup = [], [0], [], [], [0], [], [], [], []
    for h, r, c, s in streams:
        ops.extend(r.ops)
        acks.extend(r.acks)
        op_off.append(len(ops))
        evs = harness_events(h)
        gids = iter(release_groups(r, h))
        evs = [(k, next(gids) if k == 1 else a, b, w) for (k, a, b, w) in evs]
        ev.extend(evs)
        ev_off.append(len(ev))
        fin.append((h.core.offset_ns, h.core.seq, h.clock.now_ns))
        wall0.append(1_000_000_000)
        cool.append(c)
        sup.append(int(s))
    op_arr = np.zeros(len(ops), TK_OP_DTYPE)
    for i, (arg, t, cl, g) in enumerate(ops):
        op_arr[i] = (arg, t, cl, g)
    np.savez_compressed(
        os.path.join(HERE, name),
        ops=op_arr.view(np.uint8), op_off=np.asarray(op_off, np.int64), acks=np.asarray(acks, np.int32),
        events=np.asarray(ev, np.int64).reshape(-1, 4), ev_off=np.asarray(ev_off, np.int64),
        final=np.asarray(fin, np.int64), wall0=np.asarray(wall0, np.int64), cooldown=np.asarray(cool, np.int64),
        suppress=np.asarray(sup, np.uint8),
    )
    return len(ops), len(ev)


def make_barrier_golden():
    streams = []  # (h, rec, cooldown, suppress)
    orig_build = _support.CoreHarness.build
    recs = []

    def build(cooldown_ns=500_000, suppress=False):
        h = orig_build(cooldown_ns=cooldown_ns, suppress=suppress)
        recs.append((h, Recorder(h), cooldown_ns, suppress))
        return h

    _support.CoreHarness.build = staticmethod(build)
    try:
        for seed in range(1000):
            _support.run_random_schedule(seed)
        for seed in range(1000, 1100):  # other cooldowns
            _support.run_random_schedule(seed, cooldown_ns=[0, 1, 123_456_789, 2_000_000][seed % 4])
    finally:
        _support.CoreHarness.build = orig_build
    streams.extend(recs)
    h, r = scripted()
    streams.append((h, r, 500_000, False))
    for h, r in scenario_streams():
        streams.append((h, r, h.core.cooldown_ns, h.core.suppress_broadcasts))

    n_ops, n_ev = save_streams(streams, "barrier.npz")
    print("barrier:", len(streams), "streams,", n_ops, "ops,", n_ev, "events")


# ------------------------------------------------------------------------------
# BarrierCore at the actor counts the sweep configs use (6-32 clients)
# ------------------------------------------------------------------------------

WIDE_ACTORS = (6, 7, 8, 9, 9, 9, 12, 16, 17, 17, 17, 24, 31, 32, 32)
WIDE_COOLDOWNS = (0, 1, 500_000, 500_000, 2_000_000, 123_000_000)


def wide_schedule(seed, transcript=None, actor_counts=None, n_groups=4, obs_max=None):
    """One CoreHarness-driven schedule with 6-32 clients (A up to 17 and beyond).

    Unlike run_random_schedule (pkg/tests/_support.py:99, 1-5 actors), collectives here
    are sized up to every live actor ("all-hands" groups that make the whole actor set
    exempt one by one), actors jump while inside a group (exemption dropped,
    timekeeper.py:213), deregister inside an open group (timekeeper.py:294-314), and the
    error paths (observer jumps, non-positive targets, unknown ids, bad expected) are
    interleaved with real traffic. Every message goes through the reference BarrierCore.
    """
    rng = random.Random(seed)
    n_act = rng.choice(actor_counts or WIDE_ACTORS)
    if obs_max is None:
        n_obs = 0 if n_act >= 32 else rng.randint(0, min(2, 32 - n_act))
    else:
        n_obs = rng.randint(0, obs_max)
    cooldown = rng.choice(WIDE_COOLDOWNS)
    suppress = rng.random() < 0.15
    h = _support.CoreHarness.build(cooldown_ns=cooldown, suppress=suppress)
    rec = Recorder(h)
    if transcript is not None:
        transcript(h, cooldown, suppress)
    roles = ["A"] * n_act + ["O"] * n_obs
    rng.shuffle(roles)
    actors, observers = [], []
    for r in roles:
        (actors if r == "A" else observers).append(h.register_actor() if r == "A" else h.register_observer())
    h.seal()
    alive = list(actors)
    targets = {}
    groups = {}  # name -> expected size of the open round (None when closed)
    members = {}  # name -> set of arrived ids

    def fresh(cid):
        targets[cid] = h.virtual_now() + rng.randint(1, rng.choice((50_000, 5_000_000, 50_000_000)))

    def jump(cid):
        if h.virtual_now() >= targets[cid]:
            fresh(cid)
        h.jump(cid, targets[cid])

    def enter(cid, g, size):
        ack = h.enter(cid, g, size)
        if ack.error is None:
            members.setdefault(g, set()).add(cid)
            if len(members[g]) == size:
                members[g] = set()
                groups[g] = None
        return ack

    for cid in actors:
        fresh(cid)
    busy = lambda c: any(c in m for m in members.values())  # noqa: E731
    for _ in range(rng.randint(10, 25) * n_act):
        if not alive:
            break
        cid = rng.choice(alive)
        roll = rng.random()
        if roll < 0.50:
            if not busy(cid) or rng.random() < 0.1:  # a jump from inside a group drops exemption
                jump(cid)
        elif roll < 0.58:
            h.clock.advance(rng.choice((0, 1, rng.randint(1, 2_000_000))))
        elif roll < 0.70:
            g = f"g{rng.randint(0, n_groups - 1)}"
            if groups.get(g) is None:
                groups[g] = rng.choice((len(alive), rng.randint(1, len(alive))))
            size = groups[g] if rng.random() > 0.04 else groups[g] + 1  # occasional ExpectedMismatch
            enter(cid, g, size)
        elif roll < 0.73:
            # all-hands collective: every live actor enters one by one, the rest keep jumping
            g = "all"
            if groups.get(g) is None and not members.get(g):
                groups[g] = len(alive)
                order = list(alive)
                rng.shuffle(order)
                for c in order:
                    enter(c, g, groups[g])
                    for o in rng.sample(alive, min(len(alive), 3)):
                        if not busy(o):
                            jump(o)
        elif roll < 0.77 and len(alive) > 1:
            h.deregister(cid)
            alive.remove(cid)
            targets.pop(cid, None)
            for m in members.values():
                m.discard(cid)
        elif roll < 0.80:
            pick = rng.randrange(6)
            if pick == 0 and observers:
                h.jump(rng.choice(observers), targets.get(cid, 5))
            elif pick == 1:
                h.jump(cid, rng.choice((0, -5)))
            elif pick == 2:
                h.jump(f"actor{40 + rng.randrange(9)}", 5)
            elif pick == 3:
                h.enter(cid, "bad", 0)
            elif pick == 4 and len(actors) > len(alive):
                h.jump(rng.choice([a for a in actors if a not in alive]), 5)
            else:
                h.deregister(rng.choice([a for a in actors if a not in alive] or [f"actor{50}"]))
        else:
            jump(cid)
    for _ in range(12):  # drain: everyone outside a group jumps to its target
        any_ = False
        for cid in alive:
            if not busy(cid) and h.virtual_now() < targets[cid]:
                h.jump(cid, targets[cid])
                any_ = True
        if not any_:
            break
    return h, rec, cooldown, suppress


def resolve_rounds(A, C, rng, words=False):
    """Single resolve rounds for C Timekeepers of A actor slots, each computed by the
    reference BarrierCore._try_resolve/_resolve (timekeeper.py:318-366) on a FakeClock.

    Returns the bulk-resolve inputs (pending [C*A] with INT64_MAX = none, eligible
    bitmasks, offset, seq, wall, last broadcast with INT64_MIN = None) and the reference's
    outputs (broadcast flag 1 / silent 0 / unresolved -1, and the post-round state)."""
    I64MAX, I64MIN = np.iinfo(np.int64).max, np.iinfo(np.int64).min
    pend = np.full(C * A, I64MAX, np.int64)
    W = (A + 31) // 32
    elig = np.zeros((C, W), np.uint32) if words else np.zeros(C, np.uint32)
    st_in = np.zeros((C, 4), np.int64)
    st_out = np.zeros((C, 4), np.int64)
    flag = np.zeros(C, np.int8)
    cool = 500_000
    for c in range(C):
        h = _support.CoreHarness.build(cooldown_ns=cool)
        core = h.core
        ids = [h.register_actor() for _ in range(A)]
        core.sealed = True
        mask = rng.getrandbits(A) if rng.random() < 0.6 else (1 << A) - 1
        if mask == 0:
            mask = 1 << rng.randrange(A)
        kind = rng.random()
        p_below = rng.choice((0.0, 0.0, 0.02, 0.2))
        wall = 10**9 + rng.randint(0, 10**12)
        h.clock.now_ns = wall
        core.offset_ns = rng.choice((0, rng.randint(0, 10**9)))
        core.seq = rng.randint(0, 1000)
        core.last_broadcast_wall_ns = None if rng.random() < 0.3 else wall - rng.choice((0, 1, rng.randint(0, 10**6)))
        for a, cid in enumerate(ids):
            if not (mask >> a) & 1:
                core.exempt.add(cid) if rng.random() < 0.5 else setattr(core.clients[cid], "active", False)
                continue
            if kind < 0.15 and rng.random() < 0.2:
                continue  # round still open: unresolved
            lo = wall - 10**6 if rng.random() < p_below else wall + 1
            core.pending[cid] = rng.randint(max(1, lo), wall + rng.choice((1000, 10**6, 10**9)))
        for a, cid in enumerate(ids):
            if cid in core.pending:
                pend[c * A + a] = core.pending[cid]
        if words:
            elig[c] = [(mask >> (32 * k)) & 0xFFFFFFFF for k in range(W)]
        else:
            elig[c] = mask
        last = core.last_broadcast_wall_ns
        st_in[c] = (core.offset_ns, core.seq, wall, I64MIN if last is None else last)
        seq0 = core.seq
        n_pend = len(core.pending)
        core._try_resolve()
        resolved = n_pend and not core.pending
        flag[c] = -1 if not resolved else (1 if core.seq > seq0 else 0)
        last = core.last_broadcast_wall_ns
        st_out[c] = (core.offset_ns, core.seq, h.clock.now_ns, I64MIN if last is None else last)
    return pend, elig, st_in, st_out, flag


def make_wide_golden():
    streams, transcripts = [], []
    for seed in range(360):
        tr_hook = None
        if seed < 120:
            def tr_hook(h, cooldown, suppress):
                tr = {"cooldown": cooldown, "suppress": suppress, "steps": []}
                orig = h.core.handle

                def handle(msg, reply=None):
                    ack = orig(msg, reply)
                    tr["steps"].append({"msg": msg_doc(msg), "ack": msg_doc(ack)})
                    return ack

                h.core.handle = handle
                orig_adv = h.clock.advance

                def advance(ns):
                    orig_adv(ns)
                    tr["steps"].append({"advance": int(ns)})

                h.clock.advance = advance
                transcripts.append((h, tr))
        streams.append(wide_schedule(7_000 + seed, tr_hook))
    n_ops, n_ev = save_streams(streams, "barrier_wide.npz")
    acts = sorted({sum(1 for o in r.ops if o[1] == 0) for _, r, _, _ in streams})
    print("barrier_wide:", len(streams), "streams,", n_ops, "ops,", n_ev, "events; actor counts", acts)
    out = []
    for h, tr in transcripts:
        tr["records"] = h.records
        tr["emitted"] = [msg_doc(m) for m in h.broadcasts]
        tr["final"] = [h.core.offset_ns, h.core.seq, h.clock.now_ns]
        out.append(tr)
    import gzip

    with open(os.path.join(HERE, "core_log_wide.json.gz"), "wb") as raw, \
            gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as fh:  # mtime=0: byte-reproducible
        fh.write(json.dumps(out, separators=(",", ":")).encode())
    print("core_log_wide:", len(out), "transcripts,", sum(len(t["steps"]) for t in out), "messages")
    rng = random.Random(20260217)
    arrs = {}
    for A in (9, 17, 32):
        pend, elig, st_in, st_out, flag = resolve_rounds(A, 1500, rng)
        arrs |= {f"pending{A}": pend, f"elig{A}": elig, f"in{A}": st_in, f"out{A}": st_out, f"flag{A}": flag}
        print(f"resolve A={A}:", {k: int((flag == k).sum()) for k in (-1, 0, 1)})
    np.savez_compressed(os.path.join(HERE, "resolve_wide.npz"), **arrs)


XWIDE_ACTORS = (33, 40, 48, 64, 65, 100, 130, 257)


def make_resolve_xwide_golden():
    """resolve_xwide.npz: single rounds of the reference BarrierCore._resolve for A = 33,
    65 (TP8 x PP8 + dispatcher) and 257 actor slots (tw_tk_resolve_wide)."""
    rng = random.Random(20261017)
    arrs = {}
    for A in (33, 65, 257):
        pend, elig, st_in, st_out, flag = resolve_rounds(A, 600, rng, words=True)
        arrs |= {f"pending{A}": pend, f"elig{A}": elig, f"in{A}": st_in, f"out{A}": st_out, f"flag{A}": flag}
        print(f"resolve_xwide A={A}:", {k: int((flag == k).sum()) for k in (-1, 0, 1)})
    np.savez_compressed(os.path.join(HERE, "resolve_xwide.npz"), **arrs)


def make_xwide_golden():
    """barrier_xwide.npz: CoreHarness-driven schedules beyond 32 clients (33-257 actors plus
    up to 3 observers) and, in half of them, up to 48 collective groups: what
    tw_tk_replay_wide must reproduce (BarrierCore has no client limit)."""
    streams = []
    for seed in range(48):
        streams.append(wide_schedule(91_000 + seed, None, XWIDE_ACTORS, 48 if seed % 2 else 4, 3))
    n_ops, n_ev = save_streams(streams, "barrier_xwide.npz")
    acts = sorted({sum(1 for o in r.ops if o[1] == 0) for _, r, _, _ in streams})
    print("barrier_xwide:", len(streams), "streams,", n_ops, "ops,", n_ev, "events; actor counts", acts)


# ------------------------------------------------------------------------------
# oracle.simulate
# ------------------------------------------------------------------------------


def pred_spec_to_ref(spec):
    if spec["kind"] == "constant":
        return ref_pred.ConstantPredictor(spec["us"])
    if spec["kind"] == "linear":
        return ref_pred.LinearPredictor(*spec["coef"])
    return ref_pred.TablePredictor.from_csv(calibration.csv_path(*spec["table"]), allow_extrapolation=spec.get("ext", True))


def engine_doc(cfg: EngineConfig) -> dict:
    return {
        "chunk_size": cfg.chunk_size, "policy": cfg.policy.value, "max_batch_tokens": cfg.max_batch_tokens,
        "max_running": cfg.max_running, "kv_block_tokens": cfg.kv_block_tokens,
        "kv_capacity_blocks": cfg.kv_capacity_blocks, "workers_per_replica": cfg.workers_per_replica,
        "pp_stages": cfg.pp_stages,
    }


def run_ref_case(arrivals, cfg, spec, epoch=0):
    pred = pred_spec_to_ref(spec)
    order = sorted(range(len(arrivals)), key=lambda i: arrivals[i].offset_ns)
    idx = {arrivals[i].request_id: k for k, i in enumerate(order)}
    try:
        events = ref_oracle.simulate(arrivals, cfg, pred, epoch_ns=epoch)
        status = 0
    except ref_oracle.OracleStalled as exc:
        events = None
        status = 1 if "active" in str(exc) else 2
    except ref_pred.PredictorError as exc:
        events = None
        status = 3
    return events, status, idx


def oracle_case_list():
    MS = 1_000_000
    cases = []
    C = lambda **kw: EngineConfig(**{**dict(chunk_size=512, max_batch_tokens=1024, max_running=8, kv_block_tokens=16, kv_capacity_blocks=4096), **kw})  # noqa: E731
    ten = {"kind": "constant", "us": 10_000}
    cases += [
        ("single_two_tokens", [Arrival("r00000", 0, 512, 2)], C(), ten, 0),
        ("single_one_token", [Arrival("r00000", 0, 512, 1)], C(), ten, 0),
        ("chunked_prefill", [Arrival("r00000", 0, 512, 1)], C(chunk_size=256, max_batch_tokens=256), ten, 0),
        ("idle_gap", [Arrival("r00000", 0, 128, 1), Arrival("r00001", 1000 * MS, 128, 1)], C(), ten, 0),
        ("mixed_budget", [Arrival("r00000", 0, 384, 2), Arrival("r00001", 0, 384, 2)], C(max_batch_tokens=512), ten, 0),
        ("kv_gate", [Arrival("r00000", 0, 256, 1), Arrival("r00001", 0, 256, 1)], C(kv_capacity_blocks=24), ten, 0),
        ("stall", [Arrival("r00000", 0, 256, 1)], C(kv_capacity_blocks=8), ten, 0),
        ("prio", [Arrival("r00000", 0, 256, 3), Arrival("r00001", 15 * MS, 256, 1)], C(chunk_size=256, policy=SchedulingPolicy.PREFILL_PRIORITIZED), ten, 0),
        ("mixed_overlap", [Arrival("r00000", 0, 256, 3), Arrival("r00001", 15 * MS, 256, 1)], C(chunk_size=256), ten, 0),
        ("epoch", [Arrival("r00000", 0, 512, 2)], C(), ten, 5_000_000_000),
        ("deterministic40", [Arrival(f"r{i:05d}", i * 3 * MS, 128 + 32 * (i % 5), 1 + i % 7) for i in range(40)], C(max_batch_tokens=512), ten, 0),
        ("live_epoch", [Arrival(f"r{i:05d}", i * 2 * MS, 100 + i, 3) for i in range(30)], C(), ten, 1_790_000_000_000_000_000),
    ]
    # scheduler-vs-oracle workload (test_engine.py:271-285) with both policies
    spec = WorkloadSpec.from_doc({"source": "poisson", "qps": 50, "seed": 13, "num_requests": 60,
                                  "prompt_tokens": {"kind": "uniform", "low": 30, "high": 700},
                                  "output_tokens": {"kind": "uniform", "low": 1, "high": 12}})
    arr = generate_arrivals(spec)
    for pol in SchedulingPolicy:
        cases.append((f"engine_agree_{pol.value}", arr, C(chunk_size=256, max_batch_tokens=384, max_running=6, kv_capacity_blocks=256, policy=pol), ten, 0))
    # randomized small cases
    rng = random.Random(2601)
    tables = [(m, tp, pp) for m in calibration.MODELS for tp, pp in calibration.TP_PP_GRID]
    for k in range(72):
        n = rng.randint(1, 160)
        spec = WorkloadSpec.from_doc({"source": "poisson", "qps": rng.choice([2, 8, 30, 200]), "seed": 100 + k,
                                      "num_requests": n,
                                      "prompt_tokens": {"kind": "uniform", "low": 1, "high": rng.choice([64, 700, 3000])},
                                      "output_tokens": {"kind": "uniform", "low": 1, "high": rng.choice([4, 40, 300])}})
        arr = generate_arrivals(spec)
        chunk = rng.choice([16, 100, 256, 512])
        cfg = C(chunk_size=chunk, max_batch_tokens=chunk * rng.choice([1, 2, 4]), max_running=rng.choice([1, 2, 5, 32, 256]),
                kv_block_tokens=rng.choice([1, 16, 33]), kv_capacity_blocks=rng.choice([64, 300, 4096, 100000]),
                policy=rng.choice(list(SchedulingPolicy)))
        pk = rng.random()
        if pk < 0.5:
            ps = {"kind": "table", "table": list(rng.choice(tables)), "ext": True}
        elif pk < 0.8:
            ps = {"kind": "linear", "coef": [rng.uniform(100, 2000), rng.uniform(0, 3), rng.uniform(0, 60), rng.uniform(0, 0.01)]}
        else:
            ps = {"kind": "constant", "us": rng.choice([0, 1, 777, 10_000])}
        cases.append((f"random_{k}", arr, cfg, ps, rng.choice([0, 0, 12345, 10**15])))
    # a Table predictor without extrapolation can miss: prediction error case
    cases.append(("table_miss", [Arrival("r00000", 0, 5, 1)], C(), {"kind": "table", "table": ["8b", 1, 1], "ext": False}, 0))
    return cases


def full_size_cases():
    """BASELINE configs 1 and 3 and samples of the 1,024 grid: digests only."""
    out = []
    w1 = generate_arrivals(WorkloadSpec.from_doc({"source": "poisson", "qps": 8, "seed": 1, "num_requests": 1000,
                                                  "prompt_tokens": {"kind": "uniform", "low": 64, "high": 2048},
                                                  "output_tokens": {"kind": "uniform", "low": 16, "high": 256}}))
    base = dict(chunk_size=512, max_batch_tokens=2048, max_running=256, kv_block_tokens=16, kv_capacity_blocks=32768)
    out.append(("config1_8b_tp1", w1, EngineConfig(**base), {"kind": "table", "table": ["8b", 1, 1], "ext": True}, 0))
    out.append(("config2_8b_tp4", w1, EngineConfig(**base, workers_per_replica=4), {"kind": "table", "table": ["8b", 4, 1], "ext": True}, 0))
    w3 = generate_arrivals(WorkloadSpec.from_doc({"source": "poisson", "qps": 4, "seed": 1, "num_requests": 10000,
                                                  "prompt_tokens": {"kind": "uniform", "low": 64, "high": 2048},
                                                  "output_tokens": {"kind": "uniform", "low": 16, "high": 256}}))
    out.append(("config3_70b_tp4pp2", w3, EngineConfig(**base, workers_per_replica=4, pp_stages=2), {"kind": "table", "table": ["70b", 4, 2], "ext": True}, 0))
    rng = random.Random(7)
    for k in range(16):
        mbt = rng.choice([1024, 2048, 4096, 8192]); ch = rng.choice([128, 256, 512, 1024]); mr = rng.choice([32, 64, 128, 256])
        tp, pp = rng.choice(calibration.TP_PP_GRID); pol = rng.choice(list(SchedulingPolicy))
        model = "8b" if k < 12 else "70b"
        cfg = EngineConfig(chunk_size=ch, max_batch_tokens=mbt, max_running=mr, kv_block_tokens=16, kv_capacity_blocks=32768,
                           workers_per_replica=tp, pp_stages=pp, policy=pol)
        out.append((f"grid_{k}", w1, cfg, {"kind": "table", "table": [model, tp, pp], "ext": True}, 0))
    return out


def make_oracle_golden():
    records = []
    ev_blobs = []
    for name, arr, cfg, ps, epoch in oracle_case_list() + full_size_cases():
        events, status, idx = run_ref_case(arr, cfg, ps, epoch)
        full = name in {c[0] for c in oracle_case_list()}
        rec = {"name": name, "engine": engine_doc(cfg), "pred": ps, "epoch": epoch, "status": status,
               "arrivals": [[a.request_id, a.offset_ns, a.prompt_tokens, a.output_tokens] for a in arr] if full else None,
               "workload": None}
        if not full:
            rec["workload"] = {"n": len(arr), "first": [arr[0].offset_ns, arr[0].prompt_tokens, arr[0].output_tokens]}
        if events is not None:
            rec["n_events"] = len(events)
            rec["digest"] = str(digest_of_docs(events, idx))
            rec["final_ts"] = events[-1]["virtual_ts_ns"] if events else epoch
            rec["steps"] = events[-1]["step"] if events else 0
            first = {}
            fin = {}
            for e in events:
                if e["kind"] == "FIRST_TOKEN":
                    first[idx[e["request_id"]]] = e["virtual_ts_ns"]
                elif e["kind"] == "FINISHED":
                    fin[idx[e["request_id"]]] = e["virtual_ts_ns"]
            n = len(arr)
            rec["first_sha"] = hashlib.sha256(np.asarray([first.get(i, -1) for i in range(n)], np.int64).tobytes()).hexdigest()
            rec["finish_sha"] = hashlib.sha256(np.asarray([fin.get(i, -1) for i in range(n)], np.int64).tobytes()).hexdigest()
            if full:
                ev = np.zeros((len(events), 4), np.int64)
                for k, e in enumerate(events):
                    ev[k] = (idx[e["request_id"]], {"FIRST_TOKEN": 0, "OUTPUT_TOKEN": 1, "FINISHED": 2}[e["kind"]], e["virtual_ts_ns"], e["step"])
                rec["ev_index"] = len(ev_blobs)
                ev_blobs.append(ev)
        records.append(rec)
        print(f"  oracle case {name}: status {status}, events {rec.get('n_events')}")
    ev_off = np.zeros(len(ev_blobs) + 1, np.int64)
    for i, e in enumerate(ev_blobs):
        ev_off[i + 1] = ev_off[i] + len(e)
    np.savez_compressed(
        os.path.join(HERE, "oracle.npz"),
        cases=np.frombuffer(json.dumps(records).encode(), np.uint8),
        events=np.concatenate(ev_blobs) if ev_blobs else np.zeros((0, 4), np.int64),
        ev_off=ev_off,
    )
    print("oracle:", len(records), "cases")


# ------------------------------------------------------------------------------
# Timekeeper actor grid through the real BarrierCore
# ------------------------------------------------------------------------------


def ref_simulate_with_tk(arrivals, cfg, pred, epoch, cooldown):
    """oracle.simulate's loop (restated around the reference's own _plan) with virtual
    time driven by a real BarrierCore: actor 0 = dispatcher, actors 1.. = TP x PP
    workers. Returns (events, offset, seq, wall, bdigest)."""
    fc = _support.FakeClock(start_ns=epoch)
    bcasts = []
    core = BarrierCore(cooldown_ns=cooldown, emit=lambda m: bcasts.append(m) if m.type is MessageType.CLOCK_UPDATE else None,
                       clock=fc.clock, sleep=fc.sleep)
    TP, S = cfg.workers_per_replica, cfg.pp_stages
    A = 1 + TP * S

    def h(**kw):
        ack = core.handle(Message(**kw))
        assert ack.error is None, ack.error
        return ack

    ids = [h(type=MessageType.REGISTER, role="ACTOR").client_id for _ in range(A)]
    h(type=MessageType.SEAL)
    for a in range(1, A):  # park every worker (exempt) in a private never-releasing group
        h(type=MessageType.COLLECTIVE_ENTER, client_id=ids[a], group_id=f"park{a}", expected=2)
    arr_ts = sorted(a.offset_ns for a in arrivals)
    n = len(arr_ts)
    disp = [0]

    def V():
        return fc.now_ns + core.offset_ns

    def advance(stage_end, end):
        while True:
            while disp[0] < n and epoch + arr_ts[disp[0]] <= V():
                disp[0] += 1
            # (a dispatcher with no arrivals left keeps requesting a far target: it
            # never sets t_min, and its request completes the round after the TP
            # workers' requests, exactly like the model's "not eligible")
            if V() >= end:
                return
            cs = None
            if stage_end:
                cs = next(s for s in range(S) if stage_end[s] > V())
            # current-stage workers un-park by requesting; the dispatcher's request
            # (when it still has arrivals) completes the round
            if cs is not None:
                for t in range(TP):
                    h(type=MessageType.JUMP_REQUEST, client_id=ids[1 + cs * TP + t], target=stage_end[cs])
            far = 1 << 62
            h(type=MessageType.JUMP_REQUEST, client_id=ids[0], target=epoch + arr_ts[disp[0]] if disp[0] < n else far)
            if cs is not None:
                for t in range(TP):
                    h(type=MessageType.COLLECTIVE_ENTER, client_id=ids[1 + cs * TP + t], group_id=f"park{1 + cs * TP + t}", expected=2)

    # --- oracle.simulate restated around the reference's own _plan (oracle.py:60-114)
    from collections import deque

    future = deque(sorted(arrivals, key=lambda a: a.offset_ns))
    waiting, active = deque(), []
    now, step, events = epoch, 0, []
    while future or waiting or active:
        while future and epoch + future[0].offset_ns <= now:
            a = future.popleft()
            waiting.append(ref_oracle._Sim(a.request_id, a.prompt_tokens, a.output_tokens))
        batch, admitted = ref_oracle._plan(waiting, active, cfg)
        if batch.is_empty():
            if active or waiting:
                ref_oracle._diagnose_stall(waiting, active, cfg)
            now = epoch + future[0].offset_ns
            advance(None, now)
            continue
        step += 1
        d = pred.predict(batch)
        base = now
        now += d
        per = d // S
        ends = [base + per * (s + 1) for s in range(S)]
        ends[-1] = base + d
        advance(ends, now)
        for rid in admitted:
            sim = next(s for s in waiting if s.rid == rid)
            waiting.remove(sim)
            active.append(sim)
        by_id = {s.rid: s for s in active}
        finished = []
        for chunk in batch.prefill_chunks:
            sim = by_id[chunk.request_id]
            sim.done_prefill += chunk.chunk_tokens
            if sim.done_prefill >= sim.prompt:
                sim.emitted = 1
                events.append({"request_id": sim.rid, "kind": "FIRST_TOKEN", "virtual_ts_ns": now, "step": step})
                if sim.emitted >= sim.output:
                    events.append({"request_id": sim.rid, "kind": "FINISHED", "virtual_ts_ns": now, "step": step})
                    finished.append(sim)
        for slot in batch.decodes:
            sim = by_id[slot.request_id]
            sim.emitted += 1
            events.append({"request_id": sim.rid, "kind": "OUTPUT_TOKEN", "virtual_ts_ns": now, "step": step})
            if sim.emitted >= sim.output:
                events.append({"request_id": sim.rid, "kind": "FINISHED", "virtual_ts_ns": now, "step": step})
                finished.append(sim)
        for sim in finished:
            active.remove(sim)
    bd = 0
    for m in bcasts:
        bd = (bd + event_hash(m.seq, 0, 3, m.offset, 0)) & M64
    return events, core.offset_ns, core.seq, fc.now_ns, bd


def make_tkgrid_golden():
    recs = []
    w_small = generate_arrivals(WorkloadSpec.from_doc({"source": "poisson", "qps": 20, "seed": 5, "num_requests": 120,
                                                       "prompt_tokens": {"kind": "uniform", "low": 16, "high": 900},
                                                       "output_tokens": {"kind": "uniform", "low": 1, "high": 60}}))
    w1 = generate_arrivals(WorkloadSpec.from_doc({"source": "poisson", "qps": 8, "seed": 1, "num_requests": 1000,
                                                  "prompt_tokens": {"kind": "uniform", "low": 64, "high": 2048},
                                                  "output_tokens": {"kind": "uniform", "low": 16, "high": 256}}))
    grid = [
        ("tk_small_tp1", w_small, 1, 1, 0, "8b", 200_000),
        ("tk_small_tp4", w_small, 4, 1, 0, "8b", 500_000),
        ("tk_small_tp2pp2", w_small, 2, 2, 12345, "8b", 500_000),
        ("tk_small_tp8pp2_70b", w_small, 8, 2, 0, "70b", 500_000),
        ("tk_small_tp4pp2_nocool", w_small, 4, 2, 0, "8b", 0),
        ("tk_small_tp1pp2_bigcool", w_small, 1, 2, 0, "8b", 3_000_000),
        ("tk_config1_tp1", w1, 1, 1, 0, "8b", 500_000),
        ("tk_config2_tp4", w1, 4, 1, 0, "8b", 500_000),
        ("tk_config_tp4pp2", w1, 4, 2, 0, "8b", 500_000),
        # wide actor grids (round 2): more than 32 actors, and more stages than the presets'
        # tables (table_tp / table_pp name the calibration table a grid uses)
        ("tk_small_tp8pp8_wide", w_small, 8, 8, 0, "8b", 500_000, 8, 2),
        ("tk_small_tp4pp16_wide", w_small, 4, 16, 777, "70b", 200_000, 4, 2),
        ("tk_small_tp16pp4_wide", w_small, 16, 4, 0, "8b", 0, 8, 1),
        ("tk_config_tp8pp5_wide", w1, 8, 5, 0, "8b", 500_000, 8, 2),
    ]
    for name, arr, tp, pp, epoch, model, cool, *table in grid:
        cfg = EngineConfig(chunk_size=512, max_batch_tokens=2048, max_running=256, kv_block_tokens=16,
                           kv_capacity_blocks=32768, workers_per_replica=tp, pp_stages=pp)
        ttp, tpp = table if table else (tp, pp)
        pred = ref_pred.TablePredictor.from_csv(calibration.csv_path(model, ttp, tpp), allow_extrapolation=True)
        events, off, seq, wall, bd = ref_simulate_with_tk(arr, cfg, pred, epoch, cool)
        plain = ref_oracle.simulate(arr, cfg, pred, epoch_ns=epoch)
        assert events == plain, name  # the restated loop is the reference loop
        order = sorted(range(len(arr)), key=lambda i: arr[i].offset_ns)
        idx = {arr[i].request_id: k for k, i in enumerate(order)}
        rec = {"name": name, "n": len(arr), "seed": 5 if arr is w_small else 1, "tp": tp, "pp": pp,
               "epoch": epoch, "model": model, "cooldown": cool, "offset": off, "seq": seq, "wall": wall,
               "bdigest": str(bd), "digest": str(digest_of_docs(events, idx)), "n_events": len(events)}
        if table:
            rec["table_tp"], rec["table_pp"] = ttp, tpp
        recs.append(rec)
        print(f"  tk case {name}: seq {seq} offset {off} wall {wall}")
    with open(os.path.join(HERE, "tkgrid.json"), "w") as fh:
        json.dump(recs, fh, indent=1)


# ------------------------------------------------------------------------------
# arrivals
# ------------------------------------------------------------------------------


def make_arrivals_golden():
    out = {}
    specs = []
    for seed in range(1, 33):
        specs.append(("sweep_seed%d" % seed, {"source": "poisson", "qps": 8, "seed": seed, "num_requests": 1000,
                                              "prompt_tokens": {"kind": "uniform", "low": 64, "high": 2048},
                                              "output_tokens": {"kind": "uniform", "low": 16, "high": 256}}))
    specs.append(("config3", {"source": "poisson", "qps": 4, "seed": 1, "num_requests": 10000,
                              "prompt_tokens": {"kind": "uniform", "low": 64, "high": 2048},
                              "output_tokens": {"kind": "uniform", "low": 16, "high": 256}}))
    specs.append(("fixed", {"source": "poisson", "qps": 3.5, "seed": 99, "num_requests": 300, "prompt_tokens": 512, "output_tokens": 64}))
    shas = {}
    for name, doc in specs:
        arr = generate_arrivals(WorkloadSpec.from_doc(doc))
        ts = np.asarray([a.offset_ns for a in arr], np.int64)
        pr = np.asarray([a.prompt_tokens for a in arr], np.int32)
        op = np.asarray([a.output_tokens for a in arr], np.int32)
        shas[name] = {"doc": doc, "sha": hashlib.sha256(ts.tobytes() + pr.tobytes() + op.tobytes()).hexdigest()}
        if name in ("sweep_seed1", "fixed"):
            out[name + "_ts"] = ts
            out[name + "_prompt"] = pr
            out[name + "_output"] = op
    np.savez_compressed(os.path.join(HERE, "arrivals.npz"), **out)
    with open(os.path.join(HERE, "arrivals.json"), "w") as fh:
        json.dump(shas, fh, indent=1)
    print("arrivals:", len(specs), "workloads")


# ------------------------------------------------------------------------------
# full BarrierCore transcripts (native core pin)
# ------------------------------------------------------------------------------

_MSG_FIELDS = ("client_id", "role", "offset", "target", "seq", "group_id", "expected", "generation", "error")


def msg_doc(m) -> dict:
    d = {"type": m.type.value}
    for f in _MSG_FIELDS:
        v = getattr(m, f)
        if v is not None:
            d[f] = v
    return d


def make_core_golden():
    transcripts = []

    def wrap(h, cooldown, suppress):
        tr = {"cooldown": cooldown, "suppress": suppress, "steps": []}
        orig = h.core.handle

        def handle(msg, reply=None):
            ack = orig(msg, reply)
            tr["steps"].append({"msg": msg_doc(msg), "ack": msg_doc(ack)})
            return ack

        h.core.handle = handle
        orig_adv = h.clock.advance

        def advance(ns):
            orig_adv(ns)
            tr["steps"].append({"advance": int(ns)})

        h.clock.advance = advance
        transcripts.append((h, tr))

    orig_build = _support.CoreHarness.build

    def build(cooldown_ns=500_000, suppress=False):
        h = orig_build(cooldown_ns=cooldown_ns, suppress=suppress)
        wrap(h, cooldown_ns, suppress)
        return h

    _support.CoreHarness.build = staticmethod(build)
    try:
        for seed in range(150):
            _support.run_random_schedule(seed)
        for seed in range(1000, 1040):
            _support.run_random_schedule(seed, cooldown_ns=[0, 1, 123_456_789, 2_000_000][seed % 4])
        scripted()
        scenario_streams()
    finally:
        _support.CoreHarness.build = orig_build
    # malformed / error paths the schedules never take
    h = _support.CoreHarness.build(cooldown_ns=500_000)
    wrap(h, 500_000, False)
    core = h.core

    def malformed(bad):
        try:
            core.handle(bad)  # recorded by the wrapper when it returns an ack
        except Exception as exc:  # noqa: BLE001
            transcripts[-1][1]["steps"].append({"msg": msg_doc(bad), "raises": type(exc).__name__, "text": str(exc)})

    malformed(Message(type=MessageType.REGISTER, role="ROBOT"))
    for m in (Message(type=MessageType.JUMP_REQUEST, client_id="actor9", target=5),
              Message(type=MessageType.SEAL),
              Message(type=MessageType.DEREGISTER, client_id="nobody"),
              Message(type=MessageType.REGISTER, role="OBSERVER"),
              Message(type=MessageType.REGISTER, role="ACTOR"),
              Message(type=MessageType.REGISTER, role="ACTOR"),
              Message(type=MessageType.JUMP_REQUEST, client_id="observer1", target=5),
              Message(type=MessageType.JUMP_REQUEST, client_id="actor2", target=0),
              Message(type=MessageType.JUMP_REQUEST, client_id="actor2"),
              Message(type=MessageType.COLLECTIVE_ENTER, client_id="observer1", group_id="g", expected=2),
              Message(type=MessageType.COLLECTIVE_ENTER, client_id="actor2", group_id="g", expected=0),
              Message(type=MessageType.COLLECTIVE_ENTER, client_id="actor2", group_id="g"),
              Message(type=MessageType.COLLECTIVE_ENTER, client_id="actor2", group_id="g", expected=2),
              Message(type=MessageType.COLLECTIVE_ENTER, client_id="actor3", group_id="g", expected=3),
              Message(type=MessageType.SEAL),
              Message(type=MessageType.SEAL),
              Message(type=MessageType.REGISTER, role="ACTOR"),
              Message(type=MessageType.JUMP_REQUEST, client_id="actor3", target=1_500_000_000),
              Message(type=MessageType.DEREGISTER, client_id="actor2"),
              Message(type=MessageType.DEREGISTER, client_id="actor2"),
              Message(type=MessageType.JUMP_REQUEST, client_id="actor2", target=5),
              Message(type=MessageType.COLLECTIVE_ENTER, client_id="actor3", group_id="g", expected=1),
              Message(type=MessageType.DEREGISTER, client_id="observer1"),
              Message(type=MessageType.JUMP_REQUEST, client_id="actor3", target=2_000_000_000)):
        core.handle(m)
    for bad in (Message(type=MessageType.REGISTER, role="ROBOT"),  # sealed: RegistrationSealed ack
                Message(type=MessageType.CLOCK_UPDATE),
                Message(type=MessageType.COLLECTIVE_ENTER, client_id="actor3", expected=1)):
        malformed(bad)
    out = []
    for h, tr in transcripts:
        tr["records"] = h.records
        tr["emitted"] = [msg_doc(m) for m in h.broadcasts]
        tr["final"] = [h.core.offset_ns, h.core.seq, h.clock.now_ns]
        out.append(tr)
    import gzip

    with open(os.path.join(HERE, "core_log.json.gz"), "wb") as raw, \
            gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as fh:  # mtime=0: byte-reproducible
        fh.write(json.dumps(out, separators=(",", ":")).encode())
    print("core_log:", len(out), "transcripts,", sum(len(t["steps"]) for t in out), "messages")


# ------------------------------------------------------------------------------
# metrics (collect_metrics + RunReport.summary over oracle-mode event logs)
# ------------------------------------------------------------------------------


def summary_doc(s: dict) -> dict:
    """The summary's numbers, floats as exact hex strings."""
    out = {k: s[k] for k in ("num_requests", "virtual_elapsed_ns", "output_tokens")}
    out["tokens_per_virtual_s"] = float(s.get("tokens_per_virtual_s", 0.0)).hex()
    for m in ("ttft_ns", "e2e_ns", "tpot_ns"):
        if m in s:
            out[m] = {k: (float(v).hex() if k != "count" else v) for k, v in s[m].items()}
    return out


def make_metrics_golden():
    from timewarp.metrics import collect_metrics

    recs = []
    rng = random.Random(397)
    for name, arr, cfg, ps, epoch in oracle_case_list() + full_size_cases():
        events, status, idx = run_ref_case(arr, cfg, ps, epoch)
        if events is None:
            continue
        rep = collect_metrics(arr, events, epoch_ns=epoch, mode="oracle", workload_fingerprint="golden",
                              wall_elapsed_ns=0)
        recs.append({"name": name, "perm": None, "summary": summary_doc(rep.summary())})
        if len(arr) > 1 and (name.startswith("random_") or name in ("config1_8b_tp1", "deterministic40")):
            perm = list(range(len(arr)))
            rng.shuffle(perm)
            shuffled = [arr[i] for i in perm]
            rep = collect_metrics(shuffled, events, epoch_ns=epoch, mode="oracle", workload_fingerprint="golden",
                                  wall_elapsed_ns=0)
            recs.append({"name": name, "perm": perm, "summary": summary_doc(rep.summary())})
    with open(os.path.join(HERE, "metrics.json"), "w") as fh:
        json.dump(recs, fh)
    print("metrics:", len(recs), "summaries")


if __name__ == "__main__":
    which = set(sys.argv[1:]) or {"predictor", "predictor_neg", "barrier", "oracle", "tkgrid", "arrivals", "metrics",
                                  "core", "wide", "xwide"}
    rng = np.random.default_rng(20260100397)
    if "predictor" in which:
        make_predictor_golden(rng)
    if "predictor_neg" in which:
        make_predictor_neg_golden()
    if "barrier" in which:
        make_barrier_golden()
    if "arrivals" in which:
        make_arrivals_golden()
    if "oracle" in which:
        make_oracle_golden()
    if "tkgrid" in which:
        make_tkgrid_golden()
    if "metrics" in which:
        make_metrics_golden()
    if "core" in which:
        make_core_golden()
    if "wide" in which:
        make_wide_golden()
    if "xwide" in which:
        make_xwide_golden()
        make_resolve_xwide_golden()
