"""ctypes binding of libtwb200 (include/twb200.h) plus the numpy mirrors of its structs.

The shared library is built in-tree (``paper_2601_00397_b200/lib/libtwb200.so``) by
``paper_2601_00397_b200.build.build_native``. There is no CPU fallback: if the
library is missing every entry point raises :class:`NativeLibraryMissing`.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libtwb200.so")

ABI_VERSION = 2

# ---- status / code constants (twb200.h) ------------------------------------------
TW_OK, TW_EINVAL, TW_ECUDA, TW_ENOSMEM, TW_ECALLBACK = 0, 1, 2, 3, 4
TW_PRED_EMPTY_BATCH, TW_PRED_NEGATIVE, TW_PRED_TABLE_MISS, TW_PRED_BAD_DESC = -1, -2, -3, -4
TW_PRED_NAN, TW_PRED_OVERFLOW = -5, -6
TW_PSET_MAGIC = 0x54534550
TW_PRED_CONSTANT, TW_PRED_LINEAR, TW_PRED_TABLE = 0, 1, 2
TW_TABLE_HOLE = -(2**63)  # int64 grid; the int32 copy uses -1 (twb200.h)
TW_QHDR_FAST = 0x80000000

TW_OP_REGISTER_ACTOR, TW_OP_REGISTER_OBSERVER, TW_OP_SEAL, TW_OP_JUMP = 0, 1, 2, 3
TW_OP_ENTER, TW_OP_DEREGISTER, TW_OP_ADVANCE_CLOCK, TW_OP_BAD_CLIENT = 4, 5, 6, 7
ACK_NAMES = {
    0: None,
    1: "RegistrationSealed",
    2: "NoActors",
    3: "UnknownClient",
    4: "InvalidState",
    5: "RoleViolation",
    6: "InvalidDelta",
    7: "ExpectedMismatch",
    8: "EngineLimit",
}
TW_TK_MAX_CLIENTS = 32
TW_TK_MAX_CLIENTS_WIDE = 1024
TW_TK_MAX_GROUPS = 32
TW_TK_MAX_GROUPS_WIDE = 64

TW_POLICY_MIXED, TW_POLICY_PREFILL_PRIORITIZED = 0, 1
TW_SIM_TIMEKEEPER = 1
TW_SIM_OK, TW_SIM_STALLED_ACTIVE, TW_SIM_STALLED_KV = 0, 1, 2
TW_SIM_PRED_ERROR, TW_SIM_CAPACITY, TW_SIM_BAD_CONFIG = 3, 4, 5
TW_SIM_OVERFLOW_BIT = 1 << 8
TW_EV_FIRST_TOKEN, TW_EV_OUTPUT_TOKEN, TW_EV_FINISHED = 0, 1, 2
EVENT_KIND_NAMES = ("FIRST_TOKEN", "OUTPUT_TOKEN", "FINISHED")

# ---- struct mirrors ----------------------------------------------------------------
PSET_HEADER_DTYPE = np.dtype(
    [("magic", "<u4"), ("version", "<u4"), ("n_desc", "<i4"), ("total_bytes", "<i4"),
     ("core_bytes", "<i4"), ("fast_off", "<i4"), ("n_axis_sets", "<i4"), ("reserved", "<i4")]
)
PRED_DESC_DTYPE = np.dtype(
    [
        ("kind", "<i4"),
        ("allow_extrapolation", "<i4"),
        ("constant_us", "<i8"),
        ("base_us", "<f8"),
        ("per_prefill_token_us", "<f8"),
        ("per_decode_us", "<f8"),
        ("per_context_token_us", "<f8"),
        ("table_off", "<i4"),
        ("np", "<i4"),
        ("nd", "<i4"),
        ("pad", "<i4"),
    ]
)
TK_OP_DTYPE = np.dtype([("arg", "<i8"), ("type", "<i4"), ("client", "<i2"), ("group", "<i2")])
TK_EVENT_DTYPE = np.dtype(
    [("offset_ns", "<i8"), ("seq", "<i8"), ("wall_ns", "<i8"), ("kind", "<i4"), ("op_index", "<i4")]
)
TK_FINAL_DTYPE = np.dtype(
    [
        ("offset_ns", "<i8"),
        ("seq", "<i8"),
        ("wall_ns", "<i8"),
        ("rounds", "<i8"),
        ("broadcasts", "<i8"),
        ("n_events", "<i8"),
        ("status", "<i4"),
        ("pad", "<i4"),
        ("pad2", "<i8"),
    ]
)
SIM_CFG_DTYPE = np.dtype(
    [
        ("chunk_size", "<i4"),
        ("max_batch_tokens", "<i4"),
        ("max_running", "<i4"),
        ("kv_block_tokens", "<i4"),
        ("kv_capacity_blocks", "<i4"),
        ("workers_per_replica", "<i4"),
        ("pp_stages", "<i4"),
        ("policy", "<i4"),
        ("pred_id", "<i4"),
        ("workload_id", "<i4"),
        ("epoch_ns", "<i8"),
        ("tk_cooldown_ns", "<i8"),
        ("flags", "<u4"),
        ("pad", "<i4"),
    ]
)
SIM_RESULT_DTYPE = np.dtype(
    [
        ("final_now_ns", "<i8"),
        ("steps", "<i8"),
        ("events", "<i8"),
        ("digest", "<u8"),
        ("tk_seq", "<i8"),
        ("tk_offset_ns", "<i8"),
        ("tk_wall_ns", "<i8"),
        ("status", "<i4"),
        ("pred_code", "<i4"),
    ]
)
EVENT_DTYPE = np.dtype([("ts_ns", "<i8"), ("step", "<i4"), ("req_kind", "<i4")])
LATENCY_STATS_DTYPE = np.dtype(
    [("p50", "<f8"), ("p90", "<f8"), ("p99", "<f8"), ("mean", "<f8"), ("count", "<i8")]
)
RUN_METRICS_DTYPE = np.dtype(
    [
        ("num_requests", "<i8"),
        ("output_tokens", "<i8"),
        ("virtual_elapsed_ns", "<i8"),
        ("tokens_per_virtual_s", "<f8"),
        ("ttft", LATENCY_STATS_DTYPE),
        ("e2e", LATENCY_STATS_DTYPE),
        ("tpot", LATENCY_STATS_DTYPE),
        ("status", "<i4"),
        ("n_missing", "<i4"),
    ]
)
WL_SPEC_DTYPE = np.dtype(
    [
        ("state_hi", "<u8"),
        ("state_lo", "<u8"),
        ("inc_hi", "<u8"),
        ("inc_lo", "<u8"),
        ("scale", "<f8"),
        ("prompt_kind", "<i4"),
        ("prompt_a", "<i4"),
        ("prompt_b", "<i4"),
        ("output_kind", "<i4"),
        ("output_a", "<i4"),
        ("output_b", "<i4"),
        ("has_uint32", "<i4"),
        ("uinteger", "<u4"),
    ]
)
TW_TOKENS_FIXED, TW_TOKENS_UNIFORM = 0, 1
TW_METRICS_OK, TW_METRICS_INCOMPLETE, TW_METRICS_SIM_FAILED, TW_METRICS_TOO_LARGE = 0, 1, 2, 3

assert PRED_DESC_DTYPE.itemsize == 64
assert TK_OP_DTYPE.itemsize == 16
assert TK_EVENT_DTYPE.itemsize == 32
assert TK_FINAL_DTYPE.itemsize == 64
assert SIM_CFG_DTYPE.itemsize == 64
assert SIM_RESULT_DTYPE.itemsize == 64
assert EVENT_DTYPE.itemsize == 16
assert RUN_METRICS_DTYPE.itemsize == 160
assert WL_SPEC_DTYPE.itemsize == 72

# every symbol include/twb200.h declares (tests check the .so exports all of them)
EXPORTED_SYMBOLS = (
    "tw_predict_features",
    "tw_predict_batches",
    "tw_predict_one_sync",
    "tw_service_start",
    "tw_service_predict",
    "tw_service_predict_features",
    "tw_service_stop",
    "tw_selftest_division",
    "tw_tk_replay",
    "tw_tk_replay_wide",
    "tw_tk_resolve",
    "tw_tk_resolve_wide",
    "tw_sim_many",
    "tw_sim_scratch_bytes",
    "tw_sim_seg_scratch_bytes",
    "tw_sim_set_seg_stats",
    "tw_sim_set_checks",
    "tw_sim_last_launch",
    "tw_sim_last_path",
    "tw_sim_set_profile",
    "tw_metrics_many",
    "tw_metrics_scratch_bytes",
    "tw_generate_poisson",
    "tw_core_new",
    "tw_core_free",
    "tw_core_handle",
    "tw_core_try_resolve",
    "tw_core_abort",
    "tw_core_set_suppress",
    "tw_core_state",
    "tw_core_client",
    "tw_core_group",
    "tw_abi_version",
    "tw_last_error",
    "tw_launch_count",
)


class NativeLibraryMissing(RuntimeError):
    """libtwb200.so is not built; there is deliberately no CPU fallback."""


class NativeError(RuntimeError):
    """A libtwb200 call returned a non-zero status."""


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64

_SIGNATURES = {
    "tw_predict_features": (_I32, [_P, _I64, _P, _P, _P, _P, _I64, _P, _P]),
    "tw_predict_batches": (_I32, [_P, _I64, _P, _P, _P, _P, _I64, _P, _P, _P]),
    "tw_predict_one_sync": (_I32, [_P, _I64, _P, _I32, _I32, _P, _I64, _P, _P]),
    "tw_service_start": (_I32, [_P, _I64, _I32, _P]),
    "tw_service_predict": (_I32, [_P, _P, _I32, _I32, _P]),
    "tw_service_predict_features": (_I32, [_P, _I64, _I64, _I64, _I32, _P]),
    "tw_service_stop": (_I32, [_P]),
    "tw_selftest_division": (_I32, [_I64, ctypes.c_uint64, _P, _P]),
    "tw_tk_replay": (_I32, [_P, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P]),
    "tw_tk_replay_wide": (_I32, [_P, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P]),
    "tw_tk_resolve": (_I32, [_P, _P, _I32, _I32, _I64, _P, _P, _P, _P, _P, _P]),
    "tw_tk_resolve_wide": (_I32, [_P, _P, _I32, _I32, _I64, _P, _P, _P, _P, _P, _P]),
    "tw_sim_many": (
        _I32,
        [_P, _I64, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _P, _I64, _P],
    ),
    "tw_sim_scratch_bytes": (_I64, [_I32, _I32]),
    "tw_sim_seg_scratch_bytes": (_I64, [_I32, _I64]),
    "tw_sim_set_seg_stats": (_I32, [_P]),
    "tw_sim_set_checks": (_I32, [_P]),
    "tw_sim_last_launch": (_I32, [_P, _P, _P, _P]),
    "tw_sim_last_path": (_I32, []),
    "tw_sim_set_profile": (_I32, [_P]),
    "tw_metrics_many": (_I32, [_P, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _P, _I64, _P, _P]),
    "tw_metrics_scratch_bytes": (_I64, [_I32, _I32]),
    "tw_generate_poisson": (_I32, [_P, _I32, _P, _P, _P, _P, _P, _P]),
    "tw_abi_version": (_I32, []),
    "tw_last_error": (ctypes.c_char_p, []),
    "tw_launch_count": (_I64, []),
}

_lib = None
_lock = threading.Lock()


def load(path: str | None = None) -> ctypes.CDLL:
    """Load (once) and return the native library; raise loudly when it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # TWB200_LIB swaps in an A/B build of the library (scripts/); honoured only with
        # TWB200_ALLOW_LIB_OVERRIDE=1 so a stray variable cannot replace the product library
        override = os.environ.get("TWB200_LIB") if os.environ.get("TWB200_ALLOW_LIB_OVERRIDE") == "1" else None
        p = path or override or LIB_PATH
        if not os.path.exists(p):
            raise NativeLibraryMissing(
                f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the B200 path has no CPU fallback)"
            )
        lib = ctypes.CDLL(p)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.tw_abi_version() != ABI_VERSION:
            raise NativeLibraryMissing(f"{p}: ABI {lib.tw_abi_version()} != {ABI_VERSION}; rebuild")
        _lib = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc != TW_OK:
        msg = load().tw_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed (code {rc}): {msg}")


def launch_count() -> int:
    return int(load().tw_launch_count())


def last_sim_launch() -> dict:
    vals = [ctypes.c_int32() for _ in range(4)]
    load().tw_sim_last_launch(*[ctypes.byref(v) for v in vals])
    return {
        "grid": vals[0].value,
        "block": vals[1].value,
        "smem_bytes": vals[2].value,
        "slot_capacity": vals[3].value,
        "variant": ("latency", "throughput", "segments", "global-slots")[load().tw_sim_last_path() & 3],
    }
