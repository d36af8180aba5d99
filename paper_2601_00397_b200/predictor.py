"""Batch runtime predictors, B200 edition — drop-in for ``timewarp.predictor``.

Mirrors the reference plugin surface (pkg/src/timewarp/predictor.py:27-266): the
same class names, constructor arguments, ``from_csv`` loader, exception classes
and the duck-typed ``predict(batch, hw=None) -> int ns`` method, so the reference's
own ``oracle.simulate`` and ``EmulatedEngine`` accept these objects unchanged.
``predict`` accepts any object with ``prefill_chunks`` (``chunk_tokens``,
``context_len_before``) and ``decodes`` (``context_len``) — including the
reference's own ``BatchComposition``.

Every prediction is computed by libtwb200's sm_100a kernels (exact fp64, half-even
microsecond rounding, int64 ns): ``predict`` launches one fused extraction+predict
kernel for a single batch, ``predict_many`` / :func:`predict_features` run the bulk
kernels over millions of batches. There is no Python arithmetic fallback.

A :class:`PredictorSet` packs any number of predictors into the one contiguous
blob the kernels stage into shared memory with a TMA bulk copy (twb200.h).
"""

from __future__ import annotations

import csv
import ctypes
import logging
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _lib
from ._host import host_bases
from ._lib import (
    PRED_DESC_DTYPE,
    PSET_HEADER_DTYPE,
    TW_PRED_BAD_DESC,
    TW_PRED_NAN,
    TW_PRED_OVERFLOW,
    TW_PRED_CONSTANT,
    TW_PRED_EMPTY_BATCH,
    TW_PRED_LINEAR,
    TW_PRED_NEGATIVE,
    TW_PRED_TABLE,
    TW_PRED_TABLE_MISS,
    TW_PSET_MAGIC,
    TW_QHDR_FAST,
    TW_TABLE_HOLE,
)

log = logging.getLogger(__name__)

NS_PER_US = 1_000


def _host(name: str) -> tuple:
    return host_bases("predictor", name)  # predictor.py:27-44


class PredictorError(*(_host("PredictorError") or (Exception,))):
    pass


class EmptyBatch(PredictorError, *_host("EmptyBatch")):
    """Prediction requested for a batch with no work in it."""


class NegativeDuration(PredictorError, *_host("NegativeDuration")):
    """Model parameters produced a duration below zero."""


class TableMiss(PredictorError, *_host("TableMiss")):
    """Lookup key outside the calibrated range with extrapolation disabled."""


class TableParseError(PredictorError, *_host("TableParseError")):
    """Calibration file is malformed."""


@dataclass(frozen=True)
class PrefillChunk:
    request_id: str
    chunk_tokens: int
    context_len_before: int


@dataclass(frozen=True)
class DecodeSlot:
    request_id: str
    context_len: int


@dataclass(frozen=True)
class BatchComposition:
    prefill_chunks: tuple = ()
    decodes: tuple = ()

    @property
    def total_prefill_tokens(self) -> int:
        return sum(c.chunk_tokens for c in self.prefill_chunks)

    @property
    def num_decodes(self) -> int:
        return len(self.decodes)

    @property
    def total_context(self) -> int:
        return sum(c.context_len_before for c in self.prefill_chunks) + sum(
            d.context_len for d in self.decodes
        )

    def is_empty(self) -> bool:
        return not self.prefill_chunks and not self.decodes


@dataclass(frozen=True)
class HardwareSpec:
    name: str = "default"
    parameters: dict = field(default_factory=dict)


def is_code(values):
    """True where a kernel output is a TW_PRED_* code rather than a duration: durations are
    whole microseconds x 1000 (negative ones come from tables with negative rows), the
    codes are small negatives that are not multiples of 1000 (twb200.h)."""
    v = np.asarray(values)
    return (v < 0) & (v % 1000 != 0)


def raise_for_code(code: int, context: str = "") -> None:
    """Map a kernel's per-element code to the reference exception (predictor.py:27-44)."""
    if code >= 0 or code % 1000 == 0:  # a duration (negative only from a table's own rows)
        return
    if code == TW_PRED_EMPTY_BATCH:
        raise EmptyBatch("cannot predict a duration for an empty batch")
    if code == TW_PRED_NEGATIVE:
        raise NegativeDuration(f"model produced a negative duration{context}")
    if code == TW_PRED_TABLE_MISS:
        raise TableMiss(f"no calibration for {context or 'this batch'} and extrapolation is disabled")
    if code == TW_PRED_BAD_DESC:
        raise PredictorError("predictor descriptor out of range")
    if code == TW_PRED_NAN:  # the reference's int(round(nan)) (predictor.py:142)
        raise ValueError("cannot convert float NaN to integer")
    if code == TW_PRED_OVERFLOW:  # round(+-inf), or a duration past int64 ns (engine limit)
        raise OverflowError(f"predicted duration does not fit int64 nanoseconds{context}")
    raise PredictorError(f"unknown prediction code {code}")


# ---------------------------------------------------------------------------------
# predictor objects
# ---------------------------------------------------------------------------------


class _DevicePredictor:
    """Shared plumbing: a one-predictor PredictorSet and the predict entry points."""

    _pset: "PredictorSet | None" = None

    def _descriptor(self) -> np.void:  # pragma: no cover - abstract
        raise NotImplementedError

    def _table(self):
        return None

    @property
    def predictor_set(self) -> "PredictorSet":
        if self._pset is None:
            self._pset = PredictorSet([self])
        return self._pset

    def predict(self, batch, hw: HardwareSpec | None = None) -> int:
        """Returns the predicted step duration in nanoseconds (one GPU launch).

        The live engine calls this once per step (engine.py:684): one C call stages the
        slots in pinned memory, which a one-warp kernel reads and answers in place
        (zero-copy); the call polls the answer word (~20 us on a B200 box through
        Python, launch-bound). A process that only predicts can use the resident service instead
        (``predictor_set.service()``, ~6.5 us, no launch on the round trip)."""
        code = self.predictor_set.live().predict_one(batch)
        if code < 0:
            raise_for_code(code, _describe(batch))
        return code

    def predict_many(self, batches: Sequence, raise_errors: bool = True) -> np.ndarray:
        """Bulk prediction over many batch compositions in one launch."""
        out = self.predictor_set.predict_batches(batches, np.zeros(len(batches), np.int32))
        if raise_errors and len(out):
            bad = np.flatnonzero(is_code(out))
            if bad.size:
                i = int(bad[0])
                raise_for_code(int(out[i]), _describe(batches[i]))
        return out


def _describe(batch) -> str:
    try:
        p = sum(c.chunk_tokens for c in batch.prefill_chunks)
        d = len(batch.decodes)
        return f" prefill={p} decodes={d}"
    except Exception:  # pragma: no cover
        return ""


class ConstantPredictor(_DevicePredictor):
    """Every non-empty batch takes the same fixed duration (predictor.py:100-111)."""

    def __init__(self, duration_us: int) -> None:
        if duration_us < 0:
            raise NegativeDuration(f"constant duration {duration_us}us is negative")
        self.duration_us = int(duration_us)
        self._pset = None

    def _descriptor(self):
        d = np.zeros((), PRED_DESC_DTYPE)
        d["kind"] = TW_PRED_CONSTANT
        d["constant_us"] = self.duration_us
        return d


class LinearPredictor(_DevicePredictor):
    """Affine cost model (predictor.py:114-146), evaluated in exact fp64 on device."""

    def __init__(
        self,
        base_us: float,
        per_prefill_token_us: float = 0.0,
        per_decode_us: float = 0.0,
        per_context_token_us: float = 0.0,
    ) -> None:
        self.base_us = base_us
        self.per_prefill_token_us = per_prefill_token_us
        self.per_decode_us = per_decode_us
        self.per_context_token_us = per_context_token_us
        self._pset = None

    def _descriptor(self):
        d = np.zeros((), PRED_DESC_DTYPE)
        d["kind"] = TW_PRED_LINEAR
        d["base_us"] = float(self.base_us)
        d["per_prefill_token_us"] = float(self.per_prefill_token_us)
        d["per_decode_us"] = float(self.per_decode_us)
        d["per_context_token_us"] = float(self.per_context_token_us)
        return d


class TablePredictor(_DevicePredictor):
    """Calibration-table lookup over (total_prefill_tokens, num_decodes) (predictor.py:149-242).

    On device the rows become a dense [prefill-axis x decode-axis] int64 grid with
    holes, so bracketing is an axis search and the four corners are direct loads.
    """

    def __init__(self, rows: dict, allow_extrapolation: bool = False) -> None:
        if not rows:
            raise TableParseError("calibration table has no rows")
        self._rows = {(int(p), int(d)): int(v) for (p, d), v in dict(rows).items()}
        self._prefill_axis = sorted({p for p, _ in self._rows})
        self._decode_axis = sorted({d for _, d in self._rows})
        self.allow_extrapolation = allow_extrapolation
        for (p, d), v in self._rows.items():
            if not (-(2**31) <= p < 2**31 and -(2**31) <= d < 2**31):
                raise TableParseError(f"table key {(p, d)} outside the int32 range of the device grid")
            # negative values are valid rows (the reference rejects them only in from_csv):
            # predictions are then negative multiples of 1000 ns (is_code tells codes apart)
        # exactness of the int lerp numerator on device: |(b-a)*(x-lo)| < 2^53
        vals = list(self._rows.values())
        span = max(vals) - min(vals)
        gap = max(
            [b - a for a, b in zip(self._prefill_axis, self._prefill_axis[1:])]
            + [b - a for a, b in zip(self._decode_axis, self._decode_axis[1:])]
            + [1]
        )
        if span * gap >= 2**53:
            raise TableParseError("table values x axis gaps exceed the exact fp64 range (2^53)")
        self._pset = None

    @classmethod
    def from_csv(cls, path: str, allow_extrapolation: bool = False) -> "TablePredictor":
        """Load ``total_prefill_tokens,num_decodes,duration_us`` rows (predictor.py:167-192)."""
        rows: dict = {}
        with open(path, newline="") as fh:
            reader = csv.DictReader(fh)
            expected = {"total_prefill_tokens", "num_decodes", "duration_us"}
            if reader.fieldnames is None or not expected.issubset(reader.fieldnames):
                raise TableParseError(
                    f"{path}: header must contain {sorted(expected)}, got {reader.fieldnames}"
                )
            for lineno, row in enumerate(reader, start=2):
                try:
                    key = (int(row["total_prefill_tokens"]), int(row["num_decodes"]))
                    duration = int(row["duration_us"])
                except (TypeError, ValueError) as exc:
                    raise TableParseError(f"{path}:{lineno}: {exc}") from None
                if duration < 0:
                    raise NegativeDuration(f"{path}:{lineno}: duration {duration}us is negative")
                if key in rows:
                    log.warning("calibration table %s: duplicate key %s, keeping last", path, key)
                rows[key] = duration
        return cls(rows, allow_extrapolation=allow_extrapolation)

    def _descriptor(self):
        d = np.zeros((), PRED_DESC_DTYPE)
        d["kind"] = TW_PRED_TABLE
        d["allow_extrapolation"] = int(bool(self.allow_extrapolation))
        d["np"] = len(self._prefill_axis)
        d["nd"] = len(self._decode_axis)
        return d

    def _table(self):
        pax = np.asarray(self._prefill_axis, np.int32)
        dax = np.asarray(self._decode_axis, np.int32)
        grid = np.full((len(pax), len(dax)), TW_TABLE_HOLE, np.int64)
        pi = {p: i for i, p in enumerate(self._prefill_axis)}
        di = {d: i for i, d in enumerate(self._decode_axis)}
        for (p, d), v in self._rows.items():
            grid[pi[p], di[d]] = v
        return pax, dax, grid


def build_predictor(config: dict):
    """Construct a predictor from its config document (predictor.py:245-266)."""
    kind = config.get("kind")
    if kind == "constant":
        return ConstantPredictor(duration_us=config["duration_us"])
    if kind == "linear":
        return LinearPredictor(
            base_us=config.get("base_us", 0.0),
            per_prefill_token_us=config.get("per_prefill_token_us", 0.0),
            per_decode_us=config.get("per_decode_us", 0.0),
            per_context_token_us=config.get("per_context_token_us", 0.0),
        )
    if kind == "table":
        return TablePredictor.from_csv(
            config["path"], allow_extrapolation=config.get("allow_extrapolation", False)
        )
    raise PredictorError(f"unknown predictor kind {kind!r}")


# ---------------------------------------------------------------------------------
# predictor set blob + bulk entry points
# ---------------------------------------------------------------------------------


def _bitlen_lut(axis: np.ndarray) -> np.ndarray:
    """Per bit length b = 0..32 of x = v - axis[0]: (lo[b], hi[b]) = the largest index i
    with axis[i] - axis[0] <= the smallest / largest x of that bit length, so the floor
    index of v lies in [lo[b], hi[b]] (equal for power-of-two-like axes: no search).
    Stored as int16 pairs (twb200.h table layout)."""
    a = np.asarray(axis, np.int64)
    rel = a - a[0]
    lut = np.zeros((34, 2), np.int16)
    for b in range(34):
        low = 0 if b == 0 else (1 << (b - 1))
        high = 0 if b == 0 else (1 << b) - 1
        lut[b, 0] = int(np.searchsorted(rel, low, side="right")) - 1
        lut[b, 1] = int(np.searchsorted(rel, high, side="right")) - 1
    return lut


# shared-memory staging budget of the predictor kernels (predict.cu check_pset); the
# bulk-lookup section only covers the tables that fit beside the core blob
PSET_SMEM_BUDGET = 200 * 1024 - 128


def _align(n: int, a: int) -> int:
    return (n + a - 1) // a * a


def _axis_records(axis: np.ndarray) -> np.ndarray:
    """Bulk-lookup records of one axis (twb200.h): for b = bitlen(v) of v >= 0, the
    floor interval shared by every in-range v of that bit length, as {lo, hi, info, 0};
    info = interval index, or -1 when the bucket straddles several intervals."""
    a = np.asarray(axis, np.int64)
    n = len(a)
    rec = np.zeros((32, 4), np.int32)
    for b in range(32):
        low = 0 if b == 0 else (1 << (b - 1))
        high = 0 if b == 0 else (1 << b) - 1
        lo_v, hi_v = max(low, int(a[0])), min(high, int(a[-1]))
        if lo_v > hi_v:  # bucket entirely outside the axis: any v fails lo <= v <= hi
            edge = int(a[0]) if high < a[0] else int(a[-1])
            rec[b] = (edge, edge, 0, 0)
            continue
        i_lo = int(np.searchsorted(a, lo_v, side="right")) - 1
        i_hi = int(np.searchsorted(a, hi_v, side="right")) - 1
        if i_lo != i_hi:
            rec[b] = (0, 0, -1, 0)
            continue
        nxt = int(a[i_lo + 1]) if i_lo + 1 < n else int(a[i_lo])
        rec[b] = (int(a[i_lo]), nxt, i_lo, 0)
    return rec


def _quads(grid32: np.ndarray) -> np.ndarray:
    """{c[i][j], c[i+1][j], c[i][j+1], c[i+1][j+1]} per cell, indices clamped."""
    np_, nd = grid32.shape
    i1 = np.minimum(np.arange(np_) + 1, np_ - 1)
    j1 = np.minimum(np.arange(nd) + 1, nd - 1)
    q = np.empty((np_, nd, 4), np.int32)
    q[:, :, 0] = grid32
    q[:, :, 1] = grid32[i1, :]
    q[:, :, 2] = grid32[:, j1]
    q[:, :, 3] = grid32[i1][:, j1]
    return q


class PredictorSet:
    """Many predictors packed into one device blob (layout: include/twb200.h)."""

    def __init__(self, predictors: Iterable) -> None:
        self.predictors = list(predictors)
        if not self.predictors:
            raise PredictorError("a predictor set needs at least one predictor")
        n = len(self.predictors)
        descs = np.zeros(n, PRED_DESC_DTYPE)
        pool: list[bytes] = []
        off = _align(PSET_HEADER_DTYPE.itemsize + n * PRED_DESC_DTYPE.itemsize, 16)
        cursor = off
        for i, p in enumerate(self.predictors):
            descs[i] = p._descriptor()
            tab = p._table()
            if tab is not None:
                pax, dax, grid = tab
                axes = pax.tobytes() + dax.tobytes()
                axes += b"\0" * (_align(len(axes), 8) - len(axes))
                # RN(1 / axis gap) per interval (Python float division is correctly
                # rounded): the kernels divide by gaps with a multiply + FMA corrections
                rp = np.array([1.0 / float(pax[k + 1] - pax[k]) if k + 1 < len(pax) else 0.0
                               for k in range(len(pax))], np.float64)
                rd = np.array([1.0 / float(dax[k + 1] - dax[k]) if k + 1 < len(dax) else 0.0
                               for k in range(len(dax))], np.float64)
                blob = axes + grid.tobytes() + rp.tobytes() + rd.tobytes()
                blob += _bitlen_lut(pax).tobytes() + _bitlen_lut(dax).tobytes()
                # int32 copy of the grid for the bulk kernel's gathers (half the bytes;
                # holes -1): only for values in [0, 2^31), others use the int64 grid
                vals = grid[grid != TW_TABLE_HOLE]
                small = bool(vals.size and vals.min() >= 0 and vals.max() < 2**31)
                descs[i]["pad"] = 1 if small else 0
                if small:
                    blob += np.where(grid == TW_TABLE_HOLE, -1, grid).astype(np.int32).tobytes()
                blob += b"\0" * (_align(len(blob), 16) - len(blob))
                descs[i]["table_off"] = cursor
                pool.append(blob)
                cursor += len(blob)
        core = _align(cursor, 16)
        # bulk-lookup section: per-descriptor headers, deduplicated axis records, quads
        qhdr = np.zeros((n, 2), np.uint32)
        fast = bytearray(b"\0" * _align(qhdr.nbytes, 16))
        sets: dict[bytes, int] = {}

        def axis_set(axis) -> int:
            key = np.asarray(axis, np.int32).tobytes()
            if key not in sets:
                sets[key] = core + len(fast)
                fast.extend(_axis_records(axis).tobytes())
            return sets[key]

        for i, p in enumerate(self.predictors):
            tab = p._table()
            if tab is None:
                continue
            pax, dax, grid = tab
            if not (descs[i]["pad"] == 1 and pax[0] >= 0 and dax[0] >= 0
                    and len(pax) < 2**15 and len(dax) < 2**15):
                continue  # generic path only (int64-grid, negative-valued or negative-axis tables)
            need = 16 * len(pax) * len(dax) + sum(
                32 * 16 for a in (pax, dax) if np.asarray(a, np.int32).tobytes() not in sets)
            if core + len(fast) + need > PSET_SMEM_BUDGET:
                continue  # the whole blob must fit the kernels' shared-memory staging budget
            prec, drec = axis_set(pax), axis_set(dax)
            quads = core + len(fast)
            fast.extend(_quads(np.where(grid == TW_TABLE_HOLE, -1, grid).astype(np.int32)).tobytes())
            qhdr[i, 0] = (quads // 16) | ((prec // 16) << 16)
            qhdr[i, 1] = (drec // 16) | (len(dax) << 16) | TW_QHDR_FAST
        fast[: qhdr.nbytes] = qhdr.tobytes()
        total = core + _align(len(fast), 16)
        hdr = np.zeros((), PSET_HEADER_DTYPE)
        hdr["magic"] = TW_PSET_MAGIC
        hdr["version"] = 2
        hdr["n_desc"] = n
        hdr["total_bytes"] = total
        hdr["core_bytes"] = core
        hdr["fast_off"] = core
        hdr["n_axis_sets"] = len(sets)
        buf = bytearray(total)
        hs = PSET_HEADER_DTYPE.itemsize
        buf[0:hs] = hdr.tobytes()
        buf[hs : hs + descs.nbytes] = descs.tobytes()
        pos = off
        for blob in pool:
            buf[pos : pos + len(blob)] = blob
            pos += len(blob)
        buf[core : core + len(fast)] = fast
        self.blob = np.frombuffer(bytes(buf), np.uint8)
        self.core_nbytes = core
        self._dev: dict = {}

    @property
    def nbytes(self) -> int:
        return int(self.blob.size)

    def device_blob(self, device=None):
        from ._device import require_cuda, to_device

        dev = require_cuda(device)
        key = str(dev)
        if key not in self._dev:
            self._dev[key] = to_device(self.blob, dev)
        return self._dev[key]

    # -- bulk features -> ns --------------------------------------------------------
    def predict_features(self, P, D, C, desc_id, device=None, stream=None):
        """out[i] = ns for features (P, D, C) with descriptor desc_id (torch or numpy in).

        Empty batches are encoded as P == D == 0 and C < 0 (twb200.h). Returns a CUDA
        int64 tensor when given CUDA tensors, else a numpy array. With an explicit
        `stream`, the input copies, the output allocation, the kernel and the read-back all
        run on it (no cross-stream race).
        """
        from ._device import on_stream

        with on_stream(stream):
            return self._predict_features(P, D, C, desc_id, device)

    def _predict_features(self, P, D, C, desc_id, device=None, stream=None):
        import torch

        from ._device import require_cuda, stream_handle

        dev = require_cuda(device)
        host = not isinstance(P, torch.Tensor)

        def dv(x, dt):
            if isinstance(x, torch.Tensor):
                return x.to(device=dev, dtype=dt).contiguous()
            return torch.as_tensor(np.ascontiguousarray(x)).to(device=dev, dtype=dt)

        Pt, Dt, Ct = dv(P, torch.int32), dv(D, torch.int32), dv(C, torch.int64)
        It = dv(desc_id, torch.int32)
        n = Pt.numel()
        out = torch.empty(n, dtype=torch.int64, device=dev)
        blob = self.device_blob(dev)
        rc = _lib.load().tw_predict_features(
            blob.data_ptr(), self.nbytes, Pt.data_ptr(), Dt.data_ptr(), Ct.data_ptr(),
            It.data_ptr(), n, out.data_ptr(), stream_handle(stream),
        )
        _lib.check(rc, "tw_predict_features")
        return out.cpu().numpy() if host else out

    def service(self, device=None) -> "PredictorService":
        from ._device import require_cuda

        dev = require_cuda(device)
        key = ("service", str(dev))
        if key not in self._dev:
            self._dev[key] = PredictorService(self, dev)
        return self._dev[key]

    def live(self, device=None) -> "_LiveChannel":
        from ._device import require_cuda

        dev = require_cuda(device)
        key = ("live", str(dev))
        if key not in self._dev:
            self._dev[key] = _LiveChannel(self, dev)
        return self._dev[key]

    # -- CSR batches -> features -> ns ------------------------------------------------
    def predict_csr(self, off, tok, ctx, desc_id, device=None, return_features=False, stream=None):
        """CSR batches -> ns (see _predict_csr); with an explicit `stream` every copy, the
        kernel and the read-back run on that stream."""
        from ._device import on_stream

        with on_stream(stream):
            return self._predict_csr(off, tok, ctx, desc_id, device, return_features)

    def _predict_csr(self, off, tok, ctx, desc_id, device=None, return_features=False, stream=None):
        """Fused extraction + prediction over CSR batches given as arrays (torch or numpy).

        off: int64 [nb + 1]; tok / ctx: int32 per slot (tok -1 = DecodeSlot), padded to
        a multiple of 4 elements here when needed (twb200.h); desc_id: int32 [nb].
        Returns (ns [, features [nb, 3]]) as CUDA tensors for CUDA inputs, else numpy.
        """
        import torch

        from ._device import require_cuda, stream_handle

        dev = require_cuda(device)
        host = not isinstance(off, torch.Tensor)

        def dv(x, dt):
            if isinstance(x, torch.Tensor):
                return x.to(device=dev, dtype=dt).contiguous()
            return torch.as_tensor(np.ascontiguousarray(x)).to(device=dev, dtype=dt)

        t_off, t_id = dv(off, torch.int64), dv(desc_id, torch.int32)
        t_tok, t_ctx = dv(tok, torch.int32), dv(ctx, torch.int32)
        pad = (-t_tok.numel()) % 4 or (4 if t_tok.numel() == 0 else 0)
        if pad:
            z = torch.zeros(pad, dtype=torch.int32, device=dev)
            t_tok, t_ctx = torch.cat([t_tok, z]), torch.cat([t_ctx, z])
        nb = t_off.numel() - 1
        out = torch.empty(max(nb, 1), dtype=torch.int64, device=dev)
        feat = torch.empty(max(3 * nb, 3), dtype=torch.int64, device=dev) if return_features else None
        rc = _lib.load().tw_predict_batches(
            self.device_blob(dev).data_ptr(), self.nbytes, t_off.data_ptr(), t_tok.data_ptr(), t_ctx.data_ptr(),
            t_id.data_ptr(), nb, feat.data_ptr() if feat is not None else None, out.data_ptr(),
            stream_handle(stream),
        )
        _lib.check(rc, "tw_predict_batches")
        res, f = out[:nb], (feat[: 3 * nb].view(nb, 3) if feat is not None else None)
        if host:
            res = res.cpu().numpy()
            f = f.cpu().numpy() if f is not None else None
        return (res, f) if return_features else res

    def predict_batches(self, batches: Sequence, desc_id, device=None, return_features=False):
        """Fused feature extraction + prediction for reference-style batch objects."""
        import torch

        from ._device import require_cuda, stream_handle

        dev = require_cuda(device)
        off, tok, ctx = pack_batches(batches)
        nb = len(batches)
        t_off = torch.from_numpy(off).to(dev)
        t_tok = torch.from_numpy(tok).to(dev)
        t_ctx = torch.from_numpy(ctx).to(dev)
        t_id = torch.as_tensor(np.ascontiguousarray(desc_id, np.int32)).to(dev)
        out = torch.empty(max(nb, 1), dtype=torch.int64, device=dev)
        feat = torch.empty(max(3 * nb, 3), dtype=torch.int64, device=dev) if return_features else None
        blob = self.device_blob(dev)
        rc = _lib.load().tw_predict_batches(
            blob.data_ptr(), self.nbytes, t_off.data_ptr(), t_tok.data_ptr(), t_ctx.data_ptr(),
            t_id.data_ptr(), nb, feat.data_ptr() if feat is not None else None, out.data_ptr(),
            stream_handle(),
        )
        _lib.check(rc, "tw_predict_batches")
        res = out[:nb].cpu().numpy()
        if return_features:
            return res, feat[: 3 * nb].cpu().numpy().reshape(nb, 3)
        return res


class PredictorService:
    """Resident predictor service on one device (twb200.h tw_service_*): one persistent
    warp polls a mailbox in mapped pinned host memory and answers single-batch
    predictions in place. Started on first use, stopped by ``close()`` or at exit.
    One caller thread per service, like the engine loop that uses it.

    The warp runs until ``close()``: a device-wide synchronisation in the same process
    (``torch.cuda.synchronize()``, ``cudaDeviceSynchronize``) would wait for it forever,
    so use the service in processes that only predict (the live engine replica), and
    close it before synchronising the device."""

    def __init__(self, pset: "PredictorSet", device, max_slots: int = 4096) -> None:
        import atexit

        import torch

        with torch.cuda.device(device):
            self.blob = pset.device_blob(device)
            torch.cuda.synchronize(device)  # the blob is resident before the service reads it
            h = ctypes.c_void_p()
            _lib.check(_lib.load().tw_service_start(self.blob.data_ptr(), pset.nbytes, max_slots, ctypes.byref(h)),
                       "tw_service_start")
        self._h = h
        self.max_slots = max_slots
        self._buf = np.zeros(2 * max_slots, np.int32)
        self._out = ctypes.c_int64()
        self._out_ref = ctypes.byref(self._out)
        self._fn = _lib.load().tw_service_predict
        self._ffn = _lib.load().tw_service_predict_features
        atexit.register(self.close)

    def predict_one(self, batch, desc_id: int = 0) -> int:
        """One batch: its three feature sums (predictor.py:69-84, the reference's own
        properties) go to the device in one 32-byte mailbox write; the lookup runs there."""
        chunks, decodes = batch.prefill_chunks, batch.decodes
        if not chunks and not decodes:
            return TW_PRED_EMPTY_BATCH
        P = C = 0
        for c in chunks:
            P += c.chunk_tokens
            C += c.context_len_before
        for dslot in decodes:
            C += dslot.context_len
        D = len(decodes)
        if min(P, C) < 0 or max(P, D, C) >= 1 << 48:  # outside the mailbox's fields: slot request
            return self.predict_slots(batch, desc_id)
        _lib.check(self._ffn(self._h, P, D, C, desc_id, self._out_ref), "tw_service_predict_features")
        return int(self._out.value)

    def predict_slots(self, batch, desc_id: int = 0) -> int:
        """The same through the slot request: the device reads the slots and sums them."""
        chunks, decodes = batch.prefill_chunks, batch.decodes
        n = len(chunks) + len(decodes)
        if n > self.max_slots:
            raise PredictorError(f"batch of {n} slots exceeds the service's {self.max_slots}")
        buf = self._buf
        i = 0
        for c in chunks:
            buf[i] = c.chunk_tokens
            buf[n + i] = c.context_len_before
            i += 1
        for dslot in decodes:
            buf[i] = -1
            buf[n + i] = dslot.context_len
            i += 1
        _lib.check(self._fn(self._h, buf.ctypes.data, n, desc_id, self._out_ref), "tw_service_predict")
        return int(self._out.value)

    def close(self) -> None:
        h, self._h = getattr(self, "_h", None), None
        if h is not None and h.value:
            _lib.load().tw_service_stop(h)


class _LiveChannel:
    """Single-batch prediction for the live engine (engine.py:684): one C call
    (tw_predict_one_sync) stages the slots in pinned host memory, which a one-warp
    kernel reads and answers in place (zero-copy), then synchronizes the stream.
    Not thread-safe: one channel per engine thread, like the engine loop itself."""

    def __init__(self, pset: "PredictorSet", device) -> None:
        import torch

        self.pset = pset
        self.device = device
        self.blob_ptr = pset.device_blob(device).data_ptr()
        self._torch = torch
        self._alloc(256)
        self._out = ctypes.c_int64()
        self._out_ref = ctypes.byref(self._out)
        self._fn = _lib.load().tw_predict_one_sync

    def _alloc(self, cap: int) -> None:
        self.cap = cap
        self.h = self._torch.empty(8 * cap + 16, dtype=self._torch.uint8, pin_memory=True)
        self.buf = (ctypes.c_int32 * (2 * cap))()  # tok[n] | ctx[n], filled by slice assignment
        self.buf_addr = ctypes.addressof(self.buf)

    def predict_one(self, batch) -> int:
        from ._device import stream_handle

        chunks, decodes = batch.prefill_chunks, batch.decodes
        n = len(chunks) + len(decodes)
        if n > self.cap:
            self._alloc(max(2 * self.cap, n))
        buf = self.buf
        # PrefillChunk -> its tokens, DecodeSlot -> -1; then the contexts (predictor.py:69-84)
        buf[0:n] = [c.chunk_tokens for c in chunks] + [-1] * len(decodes)
        buf[n : 2 * n] = [c.context_len_before for c in chunks] + [d.context_len for d in decodes]
        hp = self.h.data_ptr()
        rc = self._fn(self.blob_ptr, self.pset.nbytes, self.buf_addr, n, 0, hp, 8 * self.cap + 16,
                      self._out_ref, stream_handle())
        _lib.check(rc, "tw_predict_one_sync")
        return int(self._out.value)


def pack_batches(batches: Sequence):
    """Reference-style batches -> CSR (offsets int64, slot tokens int32, slot ctx int32).

    Slot tokens: chunk_tokens for a PrefillChunk, -1 for a DecodeSlot (twb200.h).
    """
    off = np.zeros(len(batches) + 1, np.int64)
    toks: list[int] = []
    ctxs: list[int] = []
    for i, b in enumerate(batches):
        for c in b.prefill_chunks:
            toks.append(int(c.chunk_tokens))
            ctxs.append(int(c.context_len_before))
        for d in b.decodes:
            toks.append(-1)
            ctxs.append(int(d.context_len))
        off[i + 1] = len(toks)
    pad = (-len(toks)) % 4 or (4 if not toks else 0)  # readable to a multiple of 4 (twb200.h)
    tok = np.asarray(toks + [0] * pad, np.int32)
    ctx = np.asarray(ctxs + [0] * pad, np.int32)
    return off, tok, ctx
