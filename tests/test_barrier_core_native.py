"""NativeBarrierCore (host C++ core) vs the reference BarrierCore.

tests/golden/core_log.json.gz holds full transcripts of the reference core
(timekeeper.py:68-398) driven by its own test harness (pkg/tests/_support.py):
every message with its ack (all fields, error text included), every structured log
record, every emitted broadcast/release and the final (offset, seq, wall). Replaying
the messages through NativeBarrierCore on the same FakeClock must reproduce all of it.
"""

import gzip
import json
import os

import pytest

from paper_2601_00397_b200.barrier_core import MalformedBody, Message, MessageType, NativeBarrierCore

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "core_log.json.gz")
FIELDS = ("client_id", "role", "offset", "target", "seq", "group_id", "expected", "generation", "error")


class FakeClock:  # pkg/tests/_support.py:25-38
    def __init__(self, start_ns: int = 1_000_000_000) -> None:
        self.now_ns = start_ns

    def clock(self) -> int:
        return self.now_ns

    def sleep(self, seconds: float) -> None:
        self.now_ns += int(round(seconds * 1e9))


def doc(m) -> dict:
    d = {"type": m.type.value}
    for f in FIELDS:
        v = getattr(m, f)
        if v is not None:
            d[f] = v
    return d


def transcripts(path=GOLDEN):
    with gzip.open(path, "rt") as fh:
        return json.load(fh)


def replay(tr):
    clock = FakeClock()
    records, emitted = [], []
    core = NativeBarrierCore(cooldown_ns=tr["cooldown"], emit=emitted.append,
                             log_record=lambda r: records.append(json.loads(json.dumps(r))),
                             clock=clock.clock, sleep=clock.sleep, suppress_broadcasts=tr["suppress"])
    for k, step in enumerate(tr["steps"]):
        if "advance" in step:
            clock.now_ns += step["advance"]
            continue
        m = step["msg"]
        msg = Message(type=MessageType(m["type"]), **{f: m[f] for f in FIELDS if f in m})
        if "raises" in step:
            with pytest.raises(MalformedBody) as exc:
                core.handle(msg)
            assert str(exc.value) == step["text"]
            continue
        got = []
        ack = core.handle(msg, got.append)
        assert got == [ack]
        assert doc(ack) == step["ack"], (k, m)
    return core, clock, records, emitted


def test_native_core_reproduces_reference_transcripts():
    trs = transcripts()
    assert len(trs) >= 200
    n_msgs = 0
    for i, tr in enumerate(trs):
        core, clock, records, emitted = replay(tr)
        assert records == tr["records"], i
        assert [doc(e) for e in emitted] == tr["emitted"], i
        assert [core.offset_ns, core.seq, clock.now_ns] == tr["final"], i
        n_msgs += len(tr["steps"])
    assert n_msgs > 10_000


def test_native_core_reproduces_reference_transcripts_6_to_32_clients():
    """120 wide schedules (make_golden.wide_schedule): 6-32 clients, all-hands collectives,
    jumps from inside groups, deregisters in open groups, error paths."""
    trs = transcripts(GOLDEN.replace("core_log", "core_log_wide"))
    assert len(trs) == 120
    for i, tr in enumerate(trs):
        core, clock, records, emitted = replay(tr)
        assert records == tr["records"], i
        assert [doc(e) for e in emitted] == tr["emitted"], i
        assert [core.offset_ns, core.seq, clock.now_ns] == tr["final"], i


def test_native_core_state_views_and_stall_diagnostics():
    clock = FakeClock()
    core = NativeBarrierCore(cooldown_ns=0, clock=clock.clock, sleep=clock.sleep)
    a = core.handle(Message(MessageType.REGISTER, role="ACTOR")).client_id
    b = core.handle(Message(MessageType.REGISTER, role="ACTOR")).client_id
    o = core.handle(Message(MessageType.REGISTER, role="OBSERVER")).client_id
    assert (a, b, o) == ("actor1", "actor2", "observer3")
    core.handle(Message(MessageType.SEAL))
    assert core.sealed and core.eligible_count() == 2 and core.active_actors() == ["actor1", "actor2"]
    core.handle(Message(MessageType.JUMP_REQUEST, client_id=a, target=2_000_000_000))
    assert core.pending == {"actor1": 2_000_000_000} and core.barrier_open_since_ns == 1_000_000_000
    core.handle(Message(MessageType.COLLECTIVE_ENTER, client_id=b, group_id="tp0", expected=2))
    assert core.exempt == {"actor2"} and core.groups["tp0"].arrived == {"actor2"}
    # actor2 is exempt now, so actor1's pending request alone completed the round
    assert core.seq == 1 and core.pending == {} and core.offset_ns == 1_000_000_000
    clock.now_ns += 3_000_000_000
    st = core.stalled()
    assert st is None or "barrier" not in st
    assert core.stalled(now_ns=clock.now_ns)["collectives"]["tp0"]["arrived"] == ["actor2"]
    core.handle(Message(MessageType.DEREGISTER, client_id=b))
    assert core.clients["actor2"].active is False and core.groups["tp0"].arrived == set()


REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def _ref_core_cls():
    import sys

    if not os.path.isdir(os.path.join(REF, "timewarp")):
        pytest.skip("reference not installed under baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from timewarp.timekeeper import BarrierCore
    from timewarp.wire import Message as RefMessage
    from timewarp.wire import MessageType as RefType

    return BarrierCore, RefMessage, RefType


class _Boom(RuntimeError):
    pass


def _drive(core_cls, fail_clock_at, fail_emit, Message=Message, MessageType=MessageType):
    """Two actors, jumps that resolve; the clock raises on its n-th read (or emit raises)."""
    clock = FakeClock()
    n = [0]

    def clk():
        n[0] += 1
        if n[0] == fail_clock_at:
            raise _Boom("clock")
        return clock.clock()

    def emit(_m):
        if fail_emit:
            raise _Boom("emit")

    # with a log sink both cores read the clock for every record (without one, the native
    # core skips the reads that only stamp records)
    core = core_cls(cooldown_ns=500_000, emit=emit, clock=clk, sleep=clock.sleep, log_record=lambda r: None)
    trace = []
    msgs = [Message(MessageType.REGISTER, role="ACTOR"), Message(MessageType.REGISTER, role="ACTOR"),
            Message(MessageType.SEAL), Message(MessageType.JUMP_REQUEST, client_id="actor1", target=2_000_000_000),
            Message(MessageType.JUMP_REQUEST, client_id="actor2", target=3_000_000_000),
            Message(MessageType.JUMP_REQUEST, client_id="actor1", target=4_000_000_000),
            Message(MessageType.JUMP_REQUEST, client_id="actor2", target=4_000_000_000)]
    for m in msgs:
        try:
            core.handle(m)
            trace.append("ok")
        except _Boom as exc:
            trace.append(str(exc))
        trace.append((core.offset_ns, core.seq, core.last_broadcast_wall_ns, sorted(core.pending.items())))
    return trace


@pytest.mark.parametrize("fail_clock_at,fail_emit", [(k, False) for k in range(1, 14)] + [(0, True)])
def test_native_core_propagates_callback_exceptions_like_the_reference(fail_clock_at, fail_emit):
    """A clock or emit callback that raises: the exception reaches the caller of handle()
    and the core keeps the state changed up to that point, as the reference core does
    (ctypes trampolines store it, tw_core_abort unwinds the native call)."""
    ref_core, ref_msg, ref_type = _ref_core_cls()
    want = _drive(ref_core, fail_clock_at, fail_emit, ref_msg, ref_type)
    got = _drive(NativeBarrierCore, fail_clock_at, fail_emit)
    assert got == want


def test_native_core_suppress_broadcasts_is_live():
    """suppress_broadcasts set after construction takes effect at the next resolve."""
    clock = FakeClock()
    emitted = []
    core = NativeBarrierCore(cooldown_ns=0, emit=emitted.append, clock=clock.clock, sleep=clock.sleep)
    a = core.handle(Message(MessageType.REGISTER, role="ACTOR")).client_id
    core.handle(Message(MessageType.SEAL))
    core.handle(Message(MessageType.JUMP_REQUEST, client_id=a, target=2_000_000_000))
    core.suppress_broadcasts = True
    core.handle(Message(MessageType.JUMP_REQUEST, client_id=a, target=3_000_000_000))
    core.suppress_broadcasts = False
    core.handle(Message(MessageType.JUMP_REQUEST, client_id=a, target=4_000_000_000))
    assert [m.seq for m in emitted] == [1, 3] and core.seq == 3
