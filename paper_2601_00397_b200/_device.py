"""Device plumbing: numpy <-> CUDA tensors and the current stream handle.

PyTorch is used only for device memory, pinned host buffers and streams; every
computation runs in libtwb200's own kernels.
"""

from __future__ import annotations

import numpy as np
import torch


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 engine needs a CUDA device (no CPU fallback)")
    return torch.device(device if device is not None else "cuda")


def as_bytes(arr: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(arr)
    return a.view(np.uint8).reshape(-1)


def to_device(arr: np.ndarray, device, non_blocking: bool = False) -> torch.Tensor:
    """Copy a numpy array (plain or structured) into a new CUDA tensor.

    Structured arrays travel as raw bytes (uint8 tensors); the kernels read them
    through the C struct layouts of include/twb200.h.
    """
    a = np.ascontiguousarray(arr)
    if a.dtype.fields is not None or a.dtype == np.uint64:
        a = a.view(np.uint8).reshape(-1)
    if not a.flags.writeable:  # torch.from_numpy wants a writable buffer; the copy is host-side
        a = a.copy()
    t = torch.from_numpy(a)
    if non_blocking:
        t = t.pin_memory()
    return t.to(device, non_blocking=non_blocking)


def empty_device(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)


def to_numpy_struct(t: torch.Tensor, dtype: np.dtype, count: int) -> np.ndarray:
    raw = t.detach().cpu().numpy().view(np.uint8)[: count * dtype.itemsize]
    return raw.view(dtype).copy()


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def on_stream(stream=None):
    """Context that makes `stream` current (a no-op for None)."""
    import contextlib

    return contextlib.nullcontext() if stream is None else torch.cuda.stream(stream)


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
