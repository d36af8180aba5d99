"""ctypes wrapper of the CPU oracle (oracle/twb_oracle.c). TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs (cpu_baseline and
``--impl reference``) may import this module; the product package never does.
The oracle restates the reference (pkg/src/timewarp/predictor.py, timekeeper.py,
oracle.py) in C and is pinned by tests/golden/ (vectors produced by running the
reference itself, tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "build", "libtwb_oracle.so")

if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2601_00397_b200._lib import (  # noqa: E402  (struct layouts only)
    EVENT_DTYPE,
    RUN_METRICS_DTYPE,
    SIM_RESULT_DTYPE,
    TK_EVENT_DTYPE,
    TK_FINAL_DTYPE,
)

_lib = None
_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64


def build() -> str:
    proc = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(proc.stdout + proc.stderr)
    return LIB


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB) or os.path.exists(os.path.join(HERE, "Makefile")):
            try:
                build()  # make: a no-op when up to date
            except (OSError, RuntimeError):
                if not os.path.exists(LIB):
                    raise
        lib = ctypes.CDLL(LIB)
        lib.orc_predict_many.argtypes = [_P, _P, _P, _P, _P, _I64, _P]
        lib.orc_predict_many.restype = None
        lib.orc_tk_replay.argtypes = [_P, _P, _I32, _P, _P, _P, _P, _P, _P, _P]
        lib.orc_tk_replay.restype = None
        lib.orc_tk_resolve.argtypes = [_P, _P, _I32, _I32, _I64, _P, _P, _P, _P, _P]
        lib.orc_tk_resolve.restype = None
        lib.orc_tk_resolve_wide.argtypes = [_P, _P, _I32, _I32, _I64, _P, _P, _P, _P, _P]
        lib.orc_tk_resolve_wide.restype = None
        lib.orc_simulate.argtypes = [_P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _I64]
        lib.orc_simulate.restype = None
        lib.orc_sim_many.argtypes = [_P, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I32]
        lib.orc_sim_many.restype = None
        lib.orc_metrics.argtypes = [_I64, _P, _P, _P, _P, _I64, _P]
        lib.orc_metrics.restype = None
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def predict_many(blob: np.ndarray, P, D, C, desc_id) -> np.ndarray:
    P = np.ascontiguousarray(P, np.int32)
    D = np.ascontiguousarray(D, np.int32)
    C = np.ascontiguousarray(C, np.int64)
    I = np.ascontiguousarray(desc_id, np.int32)
    out = np.zeros(len(P), np.int64)
    load().orc_predict_many(_p(np.ascontiguousarray(blob)), _p(P), _p(D), _p(C), _p(I), len(P), _p(out))
    return out


def tk_replay(ops: np.ndarray, op_off: np.ndarray, wall0, cooldown, suppress=None, ev_cap_per_stream=4096):
    n = len(op_off) - 1
    wall0 = np.ascontiguousarray(wall0, np.int64)
    cooldown = np.ascontiguousarray(cooldown, np.int64)
    sup = None if suppress is None else np.ascontiguousarray(suppress, np.uint8)
    ack = np.zeros(max(len(ops), 1), np.int32)
    ev_off = np.arange(n + 1, dtype=np.int64) * ev_cap_per_stream
    ev = np.zeros(max(int(ev_off[-1]), 1), TK_EVENT_DTYPE)
    fin = np.zeros(n, TK_FINAL_DTYPE)
    load().orc_tk_replay(
        _p(np.ascontiguousarray(ops)), _p(np.ascontiguousarray(op_off, np.int64)), n, _p(wall0),
        _p(cooldown), _p(sup), _p(ack), _p(ev), _p(ev_off), _p(fin),
    )
    events = [ev[ev_off[s] : ev_off[s] + min(int(fin[s]["n_events"]), ev_cap_per_stream)] for s in range(n)]
    return ack[: len(ops)], events, fin


def tk_resolve_wide(pending, elig_words, A, cooldown, offset, seq, wall, last_bcast):
    """elig_words: [C, ceil(A/32)] uint32 eligibility masks."""
    n = len(elig_words)
    bc = np.zeros(n, np.int8)
    load().orc_tk_resolve_wide(_p(pending), _p(np.ascontiguousarray(elig_words, np.uint32)), n, A, cooldown,
                               _p(offset), _p(seq), _p(wall), _p(last_bcast), _p(bc))
    return bc


def tk_resolve(pending, elig, A, cooldown, offset, seq, wall, last_bcast):
    n = len(elig)
    bc = np.zeros(n, np.int8)
    load().orc_tk_resolve(_p(pending), _p(elig), n, A, cooldown, _p(offset), _p(seq), _p(wall), _p(last_bcast), _p(bc))
    return bc


def simulate_one(blob, cfg: np.ndarray, ts, prompt, output, want_events=True):
    """One config (cfg: a SIM_CFG_DTYPE record); returns (result, first, finish, events)."""
    ts = np.ascontiguousarray(ts, np.int64)
    prompt = np.ascontiguousarray(prompt, np.int32)
    output = np.ascontiguousarray(output, np.int32)
    n = len(ts)
    res = np.zeros(1, SIM_RESULT_DTYPE)
    first = np.full(max(n, 1), -1, np.int64)
    finish = np.full(max(n, 1), -1, np.int64)
    cap = int(output.astype(np.int64).sum() + n) if want_events else 0
    ev = np.zeros(max(cap, 1), EVENT_DTYPE) if want_events else None
    c = np.ascontiguousarray(np.asarray(cfg).reshape(1))
    load().orc_simulate(
        _p(np.ascontiguousarray(blob)), _p(c), n, _p(ts), _p(prompt), _p(output), _p(res), _p(first),
        _p(finish), _p(ev), cap,
    )
    events = ev[: min(int(res[0]["events"]), cap)] if want_events else None
    return res[0], first[:n], finish[:n], events


def sim_many(blob, cfgs, wl_off, ts, prompt, output, n_threads=None, per_request=False, order=None):
    cfgs = np.ascontiguousarray(cfgs)
    n = len(cfgs)
    sizes = np.diff(wl_off)[cfgs["workload_id"]] if n else np.zeros(0, np.int64)
    req_base = np.zeros(n + 1, np.int64)
    np.cumsum(sizes, out=req_base[1:])
    res = np.zeros(n, SIM_RESULT_DTYPE)
    first = finish = None
    if per_request:
        first = np.full(max(int(req_base[-1]), 1), -1, np.int64)
        finish = np.full(max(int(req_base[-1]), 1), -1, np.int64)
    nt = n_threads or os.cpu_count() or 1
    ordp = None if order is None else np.ascontiguousarray(order, np.int32)
    load().orc_sim_many(
        _p(np.ascontiguousarray(blob)), _p(cfgs), n, _p(ordp), _p(np.ascontiguousarray(wl_off, np.int64)),
        _p(np.ascontiguousarray(ts, np.int64)), _p(np.ascontiguousarray(prompt, np.int32)),
        _p(np.ascontiguousarray(output, np.int32)), _p(res), _p(req_base), _p(first), _p(finish), nt,
    )
    return res, req_base, first, finish


def extract_features(off, tok, ctx) -> np.ndarray:
    """BatchComposition totals per CSR batch (predictor.py:69-84): int64 [nb, 3] of
    P = sum of prefill chunk tokens, D = number of decode slots, C = sum of contexts."""
    off = np.asarray(off, np.int64)
    nb = len(off) - 1
    n = int(off[-1]) if nb >= 0 else 0
    tok = np.asarray(tok, np.int64)[:n]
    ctx = np.asarray(ctx, np.int64)[:n]
    seg = np.repeat(np.arange(nb), np.diff(off))
    out = np.zeros((nb, 3), np.int64)
    np.add.at(out[:, 0], seg, np.where(tok >= 0, tok, 0))
    np.add.at(out[:, 1], seg, (tok < 0).astype(np.int64))
    np.add.at(out[:, 2], seg, ctx)
    return out


def metrics(offset_ns, output, first, finish, epoch_ns: int) -> np.ndarray:
    """RunReport.summary() numbers of one oracle-mode run (one RUN_METRICS_DTYPE record)."""
    ts = np.ascontiguousarray(offset_ns, np.int64)
    op = np.ascontiguousarray(output, np.int32)
    f = np.ascontiguousarray(first, np.int64)
    g = np.ascontiguousarray(finish, np.int64)
    out = np.zeros(1, RUN_METRICS_DTYPE)
    load().orc_metrics(len(ts), _p(ts), _p(op), _p(f), _p(g), int(epoch_ns), _p(out))
    return out[0]


# ---- the event digest, restated in Python (twb200.h: tw_event_hash) ------------------
M64 = (1 << 64) - 1


def mix64(x: int) -> int:
    x &= M64
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & M64
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & M64
    x ^= x >> 31
    return x


def event_mult(req: int, kind: int) -> int:
    return mix64(req * 0xC2B2AE3D27D4EB4F + kind * 0x165667B19E3779F9 + 0x27D4EB2F165667C5) | 1


def event_hash(k: int, req: int, kind: int, ts: int, step: int) -> int:
    """twb200.h tw_event_hash (digest v2): M(req, kind) * (k*A + ts*B + step*G + 1) mod 2^64."""
    L = k * 0x9E3779B97F4A7C15 + (ts & M64) * 0xD6E8FEB86659FD93 + (step & M64) * 0xFF51AFD7ED558CCD + 1
    return (event_mult(req, kind) * L) & M64


KIND_CODE = {"FIRST_TOKEN": 0, "OUTPUT_TOKEN": 1, "FINISHED": 2}


def digest_of_docs(events: list, req_index: dict) -> int:
    """Digest of a reference event list (dicts with request_id/kind/virtual_ts_ns/step)."""
    d = 0
    for k, e in enumerate(events):
        d = (d + event_hash(k, req_index[e["request_id"]], KIND_CODE[e["kind"]], int(e["virtual_ts_ns"]), int(e["step"]))) & M64
    return d
