"""Native BarrierCore — drop-in for ``timewarp.timekeeper.BarrierCore``.

The reference's live Timekeeper funnels every decoded message through one
single-threaded protocol state machine (pkg/src/timewarp/timekeeper.py:68-398).
:class:`NativeBarrierCore` keeps that class's constructor, ``handle(msg, reply) ->
ack`` method, attributes and ``stalled()`` diagnostics, but the state machine itself
is libtwb200's host C++ core (csrc/barrier_core.cpp, ``tw_core_*`` in twb200.h):

    server.core = NativeBarrierCore(cooldown_ns=..., emit=server._broadcast,
                                    log_record=server._write_record, ...)

Messages and acks are duck-typed against the reference's ``wire.Message``: acks and
broadcasts are built with the caller's own ``Message`` / ``MessageType`` classes
(taken from the first message handled), so the server encodes them unchanged. The
local :class:`Message` / :class:`MessageType` mirrors serve callers without the
reference. Error acks carry the reference's exact ``"Name: detail"`` strings
(errors.py:63-72); malformed messages raise :class:`MalformedBody`.
"""

from __future__ import annotations

import ctypes
import enum
import struct
import time
from dataclasses import dataclass, field

from . import _lib

DEFAULT_COOLDOWN_NS = 500_000  # timekeeper.py:36 (DEFAULT_COOLDOWN_US * NS_PER_US)
STALL_AFTER_NS = 2_000_000_000  # timekeeper.py:37


class MessageType(enum.Enum):  # wire.py:39-49
    REGISTER = "REGISTER"
    REGISTER_ACK = "REGISTER_ACK"
    SEAL = "SEAL"
    JUMP_REQUEST = "JUMP_REQUEST"
    JUMP_ACK = "JUMP_ACK"
    CLOCK_UPDATE = "CLOCK_UPDATE"
    COLLECTIVE_ENTER = "COLLECTIVE_ENTER"
    COLLECTIVE_RELEASE = "COLLECTIVE_RELEASE"
    DEREGISTER = "DEREGISTER"
    SHUTDOWN = "SHUTDOWN"


class Role(enum.Enum):  # wire.py:52-54
    ACTOR = "ACTOR"
    OBSERVER = "OBSERVER"


@dataclass
class Message:  # wire.py:73-86
    type: MessageType
    client_id: str | None = None
    role: str | None = None
    offset: int | None = None
    target: int | None = None
    seq: int | None = None
    group_id: str | None = None
    expected: int | None = None
    generation: int | None = None
    error: str | None = None


class MalformedBody(Exception):
    """Frame body is not a valid protocol message (wire.py:31-32)."""


@dataclass
class _ClientView:
    client_id: str
    role: Role
    active: bool = True


@dataclass
class _GroupView:
    group_id: str
    generation: int = 0
    expected: int | None = None
    arrived: set = field(default_factory=set)
    open_since_ns: int | None = None


_MSG_CODE = {"REGISTER": 0, "SEAL": 1, "JUMP_REQUEST": 2, "COLLECTIVE_ENTER": 3, "DEREGISTER": 4}
_ROLE_CODE = {"ACTOR": 0, "OBSERVER": 1}
_ERR_NAME = {
    1: "RegistrationSealed",
    2: "NoActors",
    3: "UnknownClient",
    4: "InvalidState",
    5: "RoleViolation",
    6: "InvalidDelta",
    7: "ExpectedMismatch",
}


class _Msg(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int32), ("client", ctypes.c_int32), ("role", ctypes.c_int32),
                ("group", ctypes.c_int32), ("target", ctypes.c_int64), ("expected", ctypes.c_int64),
                ("has_target", ctypes.c_int32), ("has_expected", ctypes.c_int32)]


class _Ack(ctypes.Structure):
    _fields_ = [("error", ctypes.c_int32), ("client", ctypes.c_int32), ("group", ctypes.c_int32),
                ("resolve", ctypes.c_int32), ("offset_ns", ctypes.c_int64), ("seq", ctypes.c_int64),
                ("generation", ctypes.c_int64)]


class _Record(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("client", ctypes.c_int32), ("role", ctypes.c_int32),
                ("group", ctypes.c_int32), ("wall_ns", ctypes.c_int64), ("offset_ns", ctypes.c_int64),
                ("seq", ctypes.c_int64), ("target_ns", ctypes.c_int64), ("expected", ctypes.c_int64),
                ("generation", ctypes.c_int64), ("t_min_ns", ctypes.c_int64), ("num_actors", ctypes.c_int32),
                ("eligible", ctypes.c_int32), ("broadcast", ctypes.c_int32), ("suppressed", ctypes.c_int32),
                ("n_items", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("items", ctypes.POINTER(ctypes.c_int32)), ("item_targets", ctypes.POINTER(ctypes.c_int64))]


class _Emit(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("group", ctypes.c_int32), ("offset_ns", ctypes.c_int64),
                ("seq", ctypes.c_int64), ("generation", ctypes.c_int64)]


class _State(ctypes.Structure):
    _fields_ = [("offset_ns", ctypes.c_int64), ("seq", ctypes.c_int64),
                ("last_broadcast_wall_ns", ctypes.c_int64), ("barrier_open_since_ns", ctypes.c_int64),
                ("sealed", ctypes.c_int32), ("has_last_broadcast", ctypes.c_int32),
                ("has_barrier_open", ctypes.c_int32), ("n_clients", ctypes.c_int32),
                ("n_groups", ctypes.c_int32), ("eligible", ctypes.c_int32), ("n_pending", ctypes.c_int32),
                ("n_active_actors", ctypes.c_int32)]


_CLOCK = ctypes.CFUNCTYPE(ctypes.c_int64, ctypes.c_void_p)
_SLEEP = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_double)
_EMIT = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.POINTER(_Emit))
_LOG = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.POINTER(_Record))


def _bind(lib):
    if getattr(lib, "_tw_core_bound", False):
        return lib
    P = ctypes.c_void_p
    lib.tw_core_new.argtypes = [ctypes.c_int64, ctypes.c_int32, _CLOCK, _SLEEP, _EMIT, _LOG, P,
                                ctypes.POINTER(ctypes.c_void_p)]
    lib.tw_core_free.argtypes = [P]
    lib.tw_core_handle.argtypes = [P, ctypes.POINTER(_Msg), ctypes.POINTER(_Ack)]
    lib.tw_core_try_resolve.argtypes = [P]
    lib.tw_core_state.argtypes = [P, ctypes.POINTER(_State)]
    lib.tw_core_client.argtypes = [P, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                   ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)]
    lib.tw_core_group.argtypes = [P, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                                  ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                  ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32), ctypes.c_int32,
                                  ctypes.POINTER(ctypes.c_int32)]
    lib.tw_core_abort.argtypes = [P]
    lib.tw_core_set_suppress.argtypes = [P, ctypes.c_int32]
    for name in ("tw_core_new", "tw_core_free", "tw_core_handle", "tw_core_try_resolve", "tw_core_state",
                 "tw_core_client", "tw_core_group", "tw_core_abort", "tw_core_set_suppress"):
        getattr(lib, name).restype = ctypes.c_int32
    lib._tw_core_bound = True
    return lib


_pack_msg = struct.Struct("<iiiiqqii").pack_into  # tw_core_msg


def _value(x):
    return x.value if isinstance(x, enum.Enum) else x


class NativeBarrierCore:
    """BarrierCore (timekeeper.py:68-398) backed by libtwb200's C++ state machine."""

    def __init__(
        self,
        cooldown_ns: int = DEFAULT_COOLDOWN_NS,
        emit=None,
        log_record=None,
        clock=time.time_ns,
        sleep=time.sleep,
        suppress_broadcasts: bool = False,
    ) -> None:
        if cooldown_ns < 0:
            raise ValueError(f"cooldown must be >= 0, got {cooldown_ns}")
        self.cooldown_ns = cooldown_ns
        self._suppress = bool(suppress_broadcasts)
        self._h = None
        self._cb_exc = None  # exception raised by a host callback, re-raised after the native call
        self._emit = emit or (lambda msg: None)
        self._log = log_record
        self._clock = clock
        self._sleep = sleep
        self._msg_cls, self._type_cls = Message, MessageType
        self._jump_ack = MessageType.JUMP_ACK
        self._ids: list[str] = []  # registration index -> client id
        self._index: dict[str, int] = {}
        self._gids: list[str] = []  # group handle -> group id
        self._ghandle: dict[str, int] = {}
        self._lib = _bind(_lib.load())
        # keep the trampolines alive as long as the core
        native_clock = clock is None or clock is time.time_ns or getattr(clock, "__name__", "") == "wall_now"
        native_sleep = sleep is None or sleep is time.sleep
        if clock is None:
            self._clock = time.time_ns
        if sleep is None:
            self._sleep = time.sleep
        self._cb = (
            _CLOCK() if native_clock else _CLOCK(self._guard(lambda _u: int(self._clock()), 0)),  # NULL: realtime
            _SLEEP() if native_sleep else _SLEEP(self._guard(lambda _u, s: self._sleep(s), None)),
            _EMIT(self._guard(self._on_emit, None)),
            _LOG(self._guard(self._on_log, None)) if log_record is not None else _LOG(),  # NULL: no records
        )
        self._codes: dict = {}
        self._mbuf, self._abuf = _Msg(), _Ack()
        self._mref, self._aref = ctypes.byref(self._mbuf), ctypes.byref(self._abuf)
        self._handle_fn, self._resolve_fn = self._lib.tw_core_handle, self._lib.tw_core_try_resolve
        h = ctypes.c_void_p()
        _lib.check(self._lib.tw_core_new(int(cooldown_ns), int(bool(suppress_broadcasts)), *self._cb, None,
                                         ctypes.byref(h)), "tw_core_new")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.tw_core_free(h)
            self._h = None

    # -- callbacks -----------------------------------------------------------
    def _guard(self, fn, default):
        """ctypes cannot propagate a Python exception through C: a failing callback stores
        it and asks the core to unwind (tw_core_abort); the native call then returns
        TW_ECALLBACK and _raise_callback re-raises it, as the reference core would."""

        def tramp(*args):
            try:
                return fn(*args)
            except BaseException as exc:  # noqa: BLE001 - re-raised after the native call
                self._cb_exc = exc
                self._lib.tw_core_abort(self._h)
                return default

        return tramp

    def _raise_callback(self, rc: int) -> None:
        # a registration the failing callback interrupted still created its client (the
        # reference adds it before logging): adopt any client ids the core holds
        n = int(self._state().n_clients)
        for i in range(len(self._ids), n):
            self._id_for(i, self._client_flags(i)[0])
        exc, self._cb_exc = self._cb_exc, None
        if exc is not None:
            raise exc
        _lib.check(rc, "tw_core callback")

    @property
    def suppress_broadcasts(self) -> bool:
        return self._suppress

    @suppress_broadcasts.setter
    def suppress_broadcasts(self, value: bool) -> None:
        """Re-read at every resolve by the reference (timekeeper.py:351-363): pushed to the core."""
        self._suppress = bool(value)
        if self._h is not None:
            self._lib.tw_core_set_suppress(self._h, int(self._suppress))

    def _mk(self, name: str, **kw):
        return self._msg_cls(type=getattr(self._type_cls, name), **kw)


    def _on_emit(self, _u, ev_p) -> None:
        ev = ev_p.contents
        if ev.kind == 0:
            self._emit(self._mk("CLOCK_UPDATE", offset=int(ev.offset_ns), seq=int(ev.seq)))
        else:
            self._emit(self._mk("COLLECTIVE_RELEASE", group_id=self._gids[ev.group], generation=int(ev.generation)))

    def _on_log(self, _u, rec_p) -> None:
        r = rec_p.contents
        k = r.kind
        if k == 0:
            doc = {"event": "register", "client_id": self._id_for(r.client, r.role), "role": "ACTOR" if r.role == 0
                   else "OBSERVER", "offset_ns": r.offset_ns, "seq": r.seq, "wall_ns": r.wall_ns}
        elif k == 1:
            doc = {"event": "seal", "num_actors": r.num_actors, "wall_ns": r.wall_ns}
        elif k == 2:
            doc = {"event": "request", "client_id": self._ids[r.client], "target_ns": r.target_ns,
                   "wall_ns": r.wall_ns}
        elif k == 3:
            doc = {"event": "collective_enter", "client_id": self._ids[r.client], "group_id": self._gids[r.group],
                   "expected": r.expected, "generation": r.generation, "wall_ns": r.wall_ns}
        elif k == 4:
            doc = {"event": "collective_release", "group_id": self._gids[r.group], "generation": r.generation,
                   "members": [self._ids[r.items[i]] for i in range(r.n_items)], "wall_ns": r.wall_ns}
        elif k == 5:
            doc = {"event": "deregister", "client_id": self._ids[r.client], "wall_ns": r.wall_ns}
        elif k == 6:
            doc = {"event": "resolve", "t_min_ns": r.t_min_ns, "wall_ns": r.wall_ns,
                   "pending": {self._ids[r.items[i]]: r.item_targets[i] for i in range(r.n_items)},
                   "eligible": r.eligible, "broadcast": bool(r.broadcast)}
        else:
            doc = {"event": "broadcast", "offset_ns": r.offset_ns, "seq": r.seq, "wall_ns": r.wall_ns,
                   "suppressed": bool(r.suppressed)}
        self._log(doc)

    def _id_for(self, idx: int, role: int) -> str:
        # client ids follow the shared registration counter (timekeeper.py:161-162)
        while len(self._ids) <= idx:
            n = len(self._ids)
            cid = f"{'actor' if role == 0 else 'observer'}{n + 1}"
            self._ids.append(cid)
            self._index[cid] = n
        return self._ids[idx]

    # -- protocol -------------------------------------------------------------
    def handle(self, msg, reply=None):
        """Dispatch one inbound message, returning (and optionally sending) its ack."""
        t = msg.type
        code = self._codes.get(t)
        if code is None:
            code = self._learn_type(msg)
        cid = msg.client_id
        client = self._index.get(cid, -1) if cid else -1
        role = group = 0
        if code == 0:
            role = _ROLE_CODE.get(_value(msg.role), -1)
        elif code == 3:
            group = -1
            gid = msg.group_id
            if gid:
                group = self._ghandle.get(gid)
                if group is None:
                    group = self._ghandle[gid] = len(self._gids)
                    self._gids.append(gid)
        target, expected = msg.target, msg.expected
        _pack_msg(self._mbuf, 0, code, client, role, group, target or 0, expected or 0,
                  target is not None, expected is not None)
        a = self._abuf
        rc = self._handle_fn(self._h, self._mref, self._aref)
        if rc:
            if rc == _lib.TW_ECALLBACK:
                self._raise_callback(rc)
            if rc == _lib.TW_EINVAL:
                if code == 0:
                    raise MalformedBody(f"unknown role {msg.role!r}")
                raise MalformedBody("COLLECTIVE_ENTER missing group_id")
            _lib.check(rc, "tw_core_handle")
        if a.error:
            ack_type = {0: "REGISTER_ACK", 2: "JUMP_ACK"}.get(code, _value(t))
            ack = self._mk(ack_type, client_id=cid, error=f"{_ERR_NAME[a.error]}: {self._detail(msg, a)}")
            if reply is not None:
                reply(ack)
            return ack
        if code == 2:
            ack = self._msg_cls(type=self._jump_ack, client_id=self._ids[client])
        elif code == 0:
            ack = self._mk("REGISTER_ACK", client_id=self._id_for(a.client, role), offset=a.offset_ns, seq=a.seq)
        elif code == 1:
            ack = self._mk("SEAL", client_id=cid)
        elif code == 3:
            ack = self._mk("COLLECTIVE_ENTER", client_id=self._ids[client], group_id=msg.group_id,
                           generation=a.generation)
        else:
            ack = self._mk("DEREGISTER", client_id=self._ids[client])
        if reply is not None:
            reply(ack)
        if a.resolve:
            rc = self._resolve_fn(self._h)
            if rc:
                self._raise_callback(rc)
        return ack

    def _learn_type(self, msg) -> int:
        """First message of a wire type: remember its code; adopt the caller's classes."""
        t = msg.type
        if not isinstance(t, MessageType) and isinstance(t, enum.Enum):
            self._msg_cls, self._type_cls = type(msg), type(t)
            self._jump_ack = self._type_cls.JUMP_ACK
        code = _MSG_CODE.get(_value(t))
        if code is None:
            raise MalformedBody(f"clients may not send {_value(t)}")
        self._codes[t] = code
        return code

    def _detail(self, msg, a) -> str:
        """The reference's exception text for each protocol error (timekeeper.py:116-314)."""
        e, t = a.error, _value(msg.type)
        if e == 1:
            return "actor set already sealed; joining mid-run is rejected"
        if e == 2:
            return "cannot seal with zero registered actors"
        if e == 3:
            return f"no such client {msg.client_id!r}"
        if e == 4:
            return f"client {msg.client_id} already deregistered"
        if e == 5:
            what = "observers cannot jump" if t == "JUMP_REQUEST" else "collectives are for actors"
            return f"{msg.client_id} is an observer; {what}"
        if e == 6:
            return f"jump target must be positive, got {msg.target}"
        if msg.expected is None or msg.expected < 1:
            return f"expected must be >= 1, got {msg.expected}"
        return (f"group {msg.group_id!r} opened with expected={int(a.generation)}, "
                f"got expected={msg.expected}")

    # -- state (read-only views of the native core) ------------------------------
    def _state(self) -> _State:
        st = _State()
        self._lib.tw_core_state(self._h, ctypes.byref(st))
        return st

    @property
    def offset_ns(self) -> int:
        return int(self._state().offset_ns)

    @property
    def seq(self) -> int:
        return int(self._state().seq)

    @property
    def sealed(self) -> bool:
        return bool(self._state().sealed)

    @property
    def last_broadcast_wall_ns(self) -> int | None:
        st = self._state()
        return int(st.last_broadcast_wall_ns) if st.has_last_broadcast else None

    @property
    def barrier_open_since_ns(self) -> int | None:
        st = self._state()
        return int(st.barrier_open_since_ns) if st.has_barrier_open else None

    def _client_flags(self, i: int):
        role, flags, tgt = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
        self._lib.tw_core_client(self._h, i, ctypes.byref(role), ctypes.byref(flags), ctypes.byref(tgt))
        return role.value, flags.value, tgt.value

    @property
    def clients(self) -> dict:
        out = {}
        for i, cid in enumerate(self._ids):
            role, flags, _ = self._client_flags(i)
            out[cid] = _ClientView(cid, Role.ACTOR if role == 0 else Role.OBSERVER, bool(flags & 1))
        return out

    @property
    def pending(self) -> dict:
        out = {}
        for i, cid in enumerate(self._ids):
            _, flags, tgt = self._client_flags(i)
            if flags & 4:
                out[cid] = tgt
        return dict(sorted(out.items()))

    @property
    def exempt(self) -> set:
        return {cid for i, cid in enumerate(self._ids) if self._client_flags(i)[1] & 2}

    @property
    def groups(self) -> dict:
        out = {}
        members = (ctypes.c_int32 * max(1, len(self._ids)))()
        for g, gid in enumerate(self._gids):
            gen, exp, since = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
            flags, nm = ctypes.c_int32(), ctypes.c_int32()
            self._lib.tw_core_group(self._h, g, ctypes.byref(gen), ctypes.byref(exp), ctypes.byref(since),
                                    ctypes.byref(flags), members, len(members), ctypes.byref(nm))
            if not flags.value & 1:
                continue
            out[gid] = _GroupView(gid, int(gen.value), int(exp.value) if flags.value & 2 else None,
                                  {self._ids[members[k]] for k in range(nm.value)},
                                  int(since.value) if flags.value & 4 else None)
        return out

    def active_actors(self) -> list[str]:
        return [c.client_id for c in self.clients.values() if c.active and c.role is Role.ACTOR]

    def eligible_count(self) -> int:
        return int(self._state().eligible)

    def stalled(self, now_ns: int | None = None, after_ns: int = STALL_AFTER_NS) -> dict | None:
        """Barrier rounds or collectives open too long (timekeeper.py:370-398)."""
        now = now_ns if now_ns is not None else self._clock()
        record: dict = {}
        pending = self.pending
        since = self.barrier_open_since_ns
        if self.sealed and pending and since is not None and now - since > after_ns:
            waiting = sorted(set(self.active_actors()) - set(pending) - self.exempt)
            record["barrier"] = {"pending": pending, "waiting_for": waiting, "open_ms": (now - since) // 1_000_000}
        groups = {}
        for g in self.groups.values():
            if g.arrived and g.open_since_ns is not None and now - g.open_since_ns > after_ns:
                groups[g.group_id] = {"arrived": sorted(g.arrived), "expected": g.expected,
                                      "open_ms": (now - g.open_since_ns) // 1_000_000}
        if groups:
            record["collectives"] = groups
        return record or None
