"""Messages/s of the reference BarrierCore (Python) vs NativeBarrierCore on the same
schedule: A actors (dispatcher + TP x PP workers) each re-requesting a target every
round on a FakeClock, broadcasts captured, log records on. Build container only."""
import json
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ".")
from timewarp.timekeeper import BarrierCore  # noqa: E402
from timewarp.wire import Message, MessageType  # noqa: E402

from paper_2601_00397_b200.barrier_core import NativeBarrierCore  # noqa: E402


class FakeClock:
    def __init__(self):
        self.now_ns = 1_000_000_000

    def clock(self):
        return self.now_ns

    def sleep(self, s):
        self.now_ns += int(round(s * 1e9))


def run(cls, A, rounds, fake=True):
    clk = FakeClock()
    out, recs = [], []
    if fake:
        core = cls(cooldown_ns=500_000, emit=out.append, log_record=recs.append, clock=clk.clock, sleep=clk.sleep)
    else:  # the live server's configuration: host realtime clock, records on (cooldown 0: no real sleeps)
        core = cls(cooldown_ns=0, emit=out.append, log_record=recs.append)
    ids = [core.handle(Message(type=MessageType.REGISTER, role="ACTOR")).client_id for _ in range(A)]
    core.handle(Message(type=MessageType.SEAL))
    msgs = [[Message(type=MessageType.JUMP_REQUEST, client_id=c, target=2_000_000_000 + (r + 1) * 1_000_000 + i)
             for i, c in enumerate(ids)] for r in range(rounds)]
    t = time.perf_counter()
    for row in msgs:
        for m in row:
            core.handle(m)
    dt = time.perf_counter() - t
    return A * rounds / dt, core.seq, core.offset_ns, len(recs)


res = {}
for A in (2, 5, 9, 17, 33):
    py = run(BarrierCore, A, 3000)
    nat = run(NativeBarrierCore, A, 3000)
    assert py[1:] == nat[1:], (A, py, nat)
    pyw = run(BarrierCore, A, 3000, fake=False)
    natw = run(NativeBarrierCore, A, 3000, fake=False)
    res[A] = {"fakeclock": {"python": round(py[0]), "native": round(nat[0]), "speedup": round(nat[0] / py[0], 2)},
              "realtime": {"python": round(pyw[0]), "native": round(natw[0]), "speedup": round(natw[0] / pyw[0], 2)}}
print(json.dumps(res))
