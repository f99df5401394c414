"""Device plumbing for the per-kernel entry points: torch allocates and
moves tensors, libbang.so computes.  No compute happens in torch here."""

from __future__ import annotations

import os

import numpy as np

from .errors import BangError

_DEVICE = None


def device_index() -> int:
    """The CUDA device this process drives (``BANG_DEVICE`` or LOCAL_RANK, else 0)."""
    global _DEVICE
    if _DEVICE is None:
        _DEVICE = int(os.environ.get("BANG_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    return _DEVICE


def set_device(index: int) -> None:
    global _DEVICE
    _DEVICE = int(index)


def torch_device():
    import torch
    if not torch.cuda.is_available():
        raise BangError("no CUDA device is visible: the B200 search path has no CPU fallback")
    return torch.device("cuda", device_index())


def to_dev(a: np.ndarray):
    import torch
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        t = torch.from_numpy(a.view(np.int64))
    else:
        t = torch.from_numpy(a)
    return t.to(torch_device())


def empty(shape, dtype):
    import torch
    tdt = {np.dtype(np.float32): torch.float32, np.dtype(np.int32): torch.int32,
           np.dtype(np.int64): torch.int64, np.dtype(np.uint64): torch.int64,
           np.dtype(np.uint8): torch.uint8, np.dtype(np.uint32): torch.int32}[np.dtype(dtype)]
    return torch.empty(shape, dtype=tdt, device=torch_device())


def to_host(t, dtype=None) -> np.ndarray:
    a = t.detach().cpu().numpy()
    if dtype is not None and np.dtype(dtype) != a.dtype:
        a = a.view(dtype)
    return a


def stream():
    import torch
    return torch.cuda.current_stream(torch_device())


def pinned_empty(shape, dtype) -> np.ndarray:
    """Host array in page-locked memory (torch's caching host allocator, so
    repeated searches reuse the pages; the array keeps its block alive).
    Device->host copies into it run at PCIe speed instead of being staged
    through the driver's bounce buffers."""
    if os.environ.get("BANG_PAGEABLE_OUT") == "1":  # (measurement: the pageable baseline)
        return np.empty(shape, dtype)
    import torch
    tdt = {np.dtype(np.float32): torch.float32, np.dtype(np.int32): torch.int32,
           np.dtype(np.int64): torch.int64, np.dtype(np.uint8): torch.uint8,
           np.dtype(np.float64): torch.float64}[np.dtype(dtype)]
    return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
