"""Timekeeper min-advance on the GPU — host side.

Mirrors the reference's BarrierCore (pkg/src/timewarp/timekeeper.py:68-366) as
seen through its test harness (pkg/tests/_support.py CoreHarness): an
:class:`OpStream` records REGISTER / SEAL / JUMP_REQUEST / COLLECTIVE_ENTER /
DEREGISTER messages (and FakeClock advances) for one Timekeeper instance, and
:func:`replay_many` replays thousands of such streams in one launch of the
``tw_tk_replay`` kernel (one warp per Timekeeper: lane = client, ballot/popc for
eligible and pending counts, one int64 warp min for t_min).

:func:`resolve_round` is the bare bulk min-advance (``tw_tk_resolve``): one
_try_resolve/_resolve round for C Timekeepers x A actor slots held in HBM.

The live TimekeeperServer (sockets, threads) stays host code, as the north star
requires; these are the batched state-machine kernels behind it.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import (
    ACK_NAMES,
    TK_EVENT_DTYPE,
    TK_FINAL_DTYPE,
    TK_OP_DTYPE,
    TW_OP_ADVANCE_CLOCK,
    TW_OP_BAD_CLIENT,
    TW_OP_DEREGISTER,
    TW_OP_ENTER,
    TW_OP_JUMP,
    TW_OP_REGISTER_ACTOR,
    TW_OP_REGISTER_OBSERVER,
    TW_OP_SEAL,
    TW_TK_MAX_CLIENTS,
    TW_TK_MAX_CLIENTS_WIDE,
    TW_TK_MAX_GROUPS,
    TW_TK_MAX_GROUPS_WIDE,
)

DEFAULT_COOLDOWN_NS = 500_000  # timekeeper.py:36
FAKE_WALL0_NS = 1_000_000_000  # pkg/tests/_support.py:28


def client_index(client_id: str) -> int:
    """'actor3' / 'observer2' -> registration index 2 / 1 (timekeeper.py:162); -1 if malformed."""
    name = client_id.rstrip("0123456789")
    digits = client_id[len(name):]
    if name not in ("actor", "observer") or not digits:
        return -1
    return int(digits) - 1


@dataclass
class OpStream:
    """Message log of one Timekeeper, in the CoreHarness vocabulary."""

    cooldown_ns: int = DEFAULT_COOLDOWN_NS
    wall0_ns: int = FAKE_WALL0_NS
    suppress_broadcasts: bool = False
    ops: list = field(default_factory=list)
    _n_clients: int = 0
    _groups: dict = field(default_factory=dict)
    _ids: dict = field(default_factory=dict)  # client id -> registration index, as the core issued them
    _live_actors: set = field(default_factory=set)
    _sealed: bool = False

    def _op(self, t, arg=0, client=0, group=0):
        self.ops.append((int(arg), t, int(client), int(group)))

    def _register(self, t, role: str):
        self._op(t)
        if self._sealed:  # RegistrationSealed: no client is created (timekeeper.py:155-157)
            return None
        self._n_clients += 1
        cid = f"{role}{self._n_clients}"
        self._ids[cid] = self._n_clients - 1
        if role == "actor":
            self._live_actors.add(cid)
        return cid

    def register_actor(self) -> str | None:
        return self._register(TW_OP_REGISTER_ACTOR, "actor")

    def register_observer(self) -> str | None:
        return self._register(TW_OP_REGISTER_OBSERVER, "observer")

    def seal(self) -> None:
        self._op(TW_OP_SEAL)
        if self._live_actors:  # sealing with no active actor fails with NoActors (timekeeper.py:176-178)
            self._sealed = True

    def _client(self, client_id: str):
        """Only ids the core issued map to a client (the reference raises UnknownClient for
        anything else, e.g. 'actor01' or an observer's index under the actor prefix)."""
        c = self._ids.get(client_id or "")
        return (c, True) if c is not None else (0, False)

    def jump(self, client_id: str, target_ns: int) -> None:
        c, ok = self._client(client_id)
        self._op(TW_OP_JUMP if ok else TW_OP_BAD_CLIENT, target_ns, c)

    def enter(self, client_id: str, group: str, expected: int) -> None:
        c, ok = self._client(client_id)
        g = self._groups.setdefault(group, len(self._groups))
        if g >= TW_TK_MAX_GROUPS_WIDE:
            raise ValueError(f"more than {TW_TK_MAX_GROUPS_WIDE} collective groups in one stream")
        self._op(TW_OP_ENTER if ok else TW_OP_BAD_CLIENT, expected, c, g)

    def deregister(self, client_id: str) -> None:
        c, ok = self._client(client_id)
        self._op(TW_OP_DEREGISTER if ok else TW_OP_BAD_CLIENT, 0, c)
        self._live_actors.discard(client_id)

    def advance(self, ns: int) -> None:
        """FakeClock.advance (pkg/tests/_support.py:36-37)."""
        self._op(TW_OP_ADVANCE_CLOCK, ns)

    def group_names(self) -> list:
        return sorted(self._groups, key=self._groups.get)


def pack_streams(streams: Sequence[OpStream]):
    ops = np.zeros(sum(len(s.ops) for s in streams), TK_OP_DTYPE)
    op_off = np.zeros(len(streams) + 1, np.int64)
    i = 0
    for k, s in enumerate(streams):
        for arg, t, c, g in s.ops:
            ops[i] = (arg, t, c, g)
            i += 1
        op_off[k + 1] = i
    wall0 = np.asarray([s.wall0_ns for s in streams], np.int64)
    cool = np.asarray([s.cooldown_ns for s in streams], np.int64)
    sup = np.asarray([int(s.suppress_broadcasts) for s in streams], np.uint8)
    return ops, op_off, wall0, cool, sup


@dataclass
class ReplayResult:
    acks: np.ndarray  # int32 per op (0 ok, else an error code, see ack_name)
    events: list  # per stream: TK_EVENT_DTYPE array (kind 0 CLOCK_UPDATE, 1 RELEASE)
    final: np.ndarray  # TK_FINAL_DTYPE per stream

    def broadcast_sequence(self, s: int) -> list:
        e = self.events[s]
        e = e[e["kind"] == 0]
        return list(zip(e["offset_ns"].tolist(), e["seq"].tolist()))


def ack_name(code: int):
    return ACK_NAMES.get(int(code), f"code{code}")


def replay_arrays(ops, op_off, wall0, cooldown, suppress=None, ev_cap_per_stream=4096, device=None,
                  wide: bool = False) -> ReplayResult:
    """Replay packed op streams on the GPU (tw_tk_replay; tw_tk_replay_wide for streams with
    more than 32 clients or groups)."""
    import torch

    from ._device import require_cuda, stream_handle, to_device, to_numpy_struct

    dev = require_cuda(device)
    n = len(op_off) - 1
    if n == 0:
        return ReplayResult(np.zeros(0, np.int32), [], np.zeros(0, TK_FINAL_DTYPE))
    d_ops = to_device(np.ascontiguousarray(ops), dev)
    d_off = to_device(np.ascontiguousarray(op_off, np.int64), dev)
    d_w = to_device(np.ascontiguousarray(wall0, np.int64), dev)
    d_c = to_device(np.ascontiguousarray(cooldown, np.int64), dev)
    d_s = to_device(np.ascontiguousarray(suppress, np.uint8), dev) if suppress is not None else None
    n_ops = int(op_off[-1])
    d_ack = torch.zeros(max(n_ops, 1), dtype=torch.int32, device=dev)
    ev_off = np.arange(n + 1, dtype=np.int64) * ev_cap_per_stream
    d_evoff = to_device(ev_off, dev)
    d_ev = torch.zeros(max(int(ev_off[-1]), 1) * TK_EVENT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    d_fin = torch.zeros(n * TK_FINAL_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    lib = _lib.load()
    fn = lib.tw_tk_replay_wide if wide else lib.tw_tk_replay
    rc = fn(
        d_ops.data_ptr(), d_off.data_ptr(), n, d_w.data_ptr(), d_c.data_ptr(),
        d_s.data_ptr() if d_s is not None else None, d_ack.data_ptr(), d_ev.data_ptr(), d_evoff.data_ptr(),
        d_fin.data_ptr(), stream_handle(),
    )
    _lib.check(rc, "tw_tk_replay_wide" if wide else "tw_tk_replay")
    fin = to_numpy_struct(d_fin, TK_FINAL_DTYPE, n)
    ev = to_numpy_struct(d_ev, TK_EVENT_DTYPE, int(ev_off[-1]))
    events = [ev[ev_off[s] : ev_off[s] + min(int(fin[s]["n_events"]), ev_cap_per_stream)] for s in range(n)]
    return ReplayResult(d_ack[:n_ops].cpu().numpy(), events, fin)


def replay_many(streams: Sequence[OpStream], ev_cap_per_stream: int = 4096, device=None) -> ReplayResult:
    """Replay op streams; streams beyond 32 clients or groups take the wide kernel."""
    ops, op_off, wall0, cool, sup = pack_streams(streams)
    for s in streams:
        if s._n_clients > TW_TK_MAX_CLIENTS_WIDE:
            raise ValueError(f"more than {TW_TK_MAX_CLIENTS_WIDE} clients in one Timekeeper stream")
    wide = any(s._n_clients > TW_TK_MAX_CLIENTS or len(s._groups) > TW_TK_MAX_GROUPS for s in streams)
    return replay_arrays(ops, op_off, wall0, cool, sup, ev_cap_per_stream, device, wide=wide)


def resolve_round_wide(pending, eligible_words, A: int, cooldown_ns: int, offset, seq, wall, last_bcast,
                       stream=None):
    """resolve_round for any A: eligible_words is a [C, ceil(A/32)] int32 tensor of masks
    (tw_tk_resolve_wide, one warp per Timekeeper)."""
    import torch

    from ._device import stream_handle

    C = eligible_words.shape[0]
    out = torch.empty(C, dtype=torch.int8, device=pending.device)
    rc = _lib.load().tw_tk_resolve_wide(
        pending.data_ptr(), eligible_words.data_ptr(), C, A, cooldown_ns, offset.data_ptr(), seq.data_ptr(),
        wall.data_ptr(), last_bcast.data_ptr(), out.data_ptr(), stream_handle(stream),
    )
    _lib.check(rc, "tw_tk_resolve_wide")
    return out


def resolve_round(pending, eligible_mask, A: int, cooldown_ns: int, offset, seq, wall, last_bcast, stream=None):
    """One bulk min-advance round over CUDA int64 tensors (updated in place).

    pending: [C*A] (INT64_MAX = no request); eligible_mask: [C] int32 bitmasks;
    last_bcast: INT64_MIN = None. Returns the int8 broadcast flags tensor
    (1 broadcast, 0 silent resolve, -1 unresolved).
    """
    import torch

    from ._device import stream_handle

    C = eligible_mask.numel()
    out = torch.empty(C, dtype=torch.int8, device=pending.device)
    rc = _lib.load().tw_tk_resolve(
        pending.data_ptr(), eligible_mask.data_ptr(), C, A, cooldown_ns, offset.data_ptr(), seq.data_ptr(),
        wall.data_ptr(), last_bcast.data_ptr(), out.data_ptr(), stream_handle(stream),
    )
    _lib.check(rc, "tw_tk_resolve")
    return out
