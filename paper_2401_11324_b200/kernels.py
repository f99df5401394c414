"""Packed (distance, id) keys, row sort and rank merge (kernels.py:1-151).

``pack_keys``/``unpack_keys`` are host bit manipulation; ``merge_sort_rows``
and ``merge_rows`` run on the GPU (kernels 4a/4b of libbang.so).
"""

from __future__ import annotations

import numpy as np

from . import _dev, _lib
from .errors import ParameterError

SENTINEL = np.uint64(0xFFFFFFFFFFFFFFFF)
_ID_MASK = np.uint64(0xFFFFFFFF)


def pack_keys(dists, ids) -> np.ndarray:
    """kernels.py:25-29: f32 bits in the high word, id in the low word."""
    d = np.ascontiguousarray(dists, dtype=np.float32)
    return (d.view(np.uint32).astype(np.uint64) << np.uint64(32)) | np.asarray(ids, dtype=np.uint64)


def unpack_keys(keys):
    """kernels.py:32-37: returns (dists float32, ids int64)."""
    keys = np.asarray(keys, dtype=np.uint64)
    ids = (keys & _ID_MASK).astype(np.int64)
    dists = (keys >> np.uint64(32)).astype(np.uint32).view(np.float32)
    return dists, ids


def _next_pow2(value: int) -> int:
    return 1 if value <= 1 else 1 << (value - 1).bit_length()


def merge_sort_rows(keys: np.ndarray) -> np.ndarray:
    """kernels.py:94-109 on the GPU: every row ascending (width a power of two)."""
    keys = np.asarray(keys, dtype=np.uint64)
    n, w = keys.shape
    if w & (w - 1):
        raise ParameterError(f"row width {w} must be a power of two")
    return sort_rows(keys)


def sort_rows(keys: np.ndarray) -> np.ndarray:
    """Any-width ascending row sort (kernel 4a)."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    n, w = keys.shape
    if n == 0 or w == 0:
        return keys.copy()
    d = _dev.to_dev(keys)
    _lib.check(_lib.lib().bang_sort_rows_device(_lib.ptr(d), n, w, _lib.stream_ptr(_dev.stream())),
               "sort_rows")
    return _dev.to_host(d, np.uint64)


def merge_rows(a_keys, b_keys, a_payload=None):
    """kernels.py:68-87 on the GPU: row-wise merge, a first on ties."""
    a = np.ascontiguousarray(a_keys, dtype=np.uint64)
    b = np.ascontiguousarray(b_keys, dtype=np.uint64)
    n, wa = a.shape
    wb = b.shape[1]
    if n == 0 or wa + wb == 0:
        out = np.empty((n, wa + wb), np.uint64)
        return out if a_payload is None else (out, np.zeros((n, wa + wb), bool))
    da, db = _dev.to_dev(a), _dev.to_dev(b)
    dout = _dev.empty((n, wa + wb), np.uint64)
    dpay = _dev.to_dev(np.ascontiguousarray(a_payload, dtype=np.uint8)) if a_payload is not None else None
    dopay = _dev.empty((n, wa + wb), np.uint8) if a_payload is not None else None
    _lib.check(_lib.lib().bang_merge_rows_device(_lib.ptr(da), _lib.ptr(dpay), n, wa, _lib.ptr(db), wb,
                                                 _lib.ptr(dout), _lib.ptr(dopay),
                                                 _lib.stream_ptr(_dev.stream())), "merge_rows")
    out = _dev.to_host(dout, np.uint64)
    if a_payload is None:
        return out
    return out, _dev.to_host(dopay).astype(bool)


def _check_sorted_pairs(items, name):
    keys = [(np.float32(d), int(i)) for i, d in items]
    if any(keys[j] > keys[j + 1] for j in range(len(keys) - 1)):
        raise ParameterError(f"{name} must be sorted by (dist, node_id)")


def parallel_merge(a, b):
    """kernels.py:112-130: merge two (id, dist) lists sorted by (dist, id)."""
    _check_sorted_pairs(a, "a")
    _check_sorted_pairs(b, "b")
    if not a:
        return [(int(i), np.float32(d)) for i, d in b]
    if not b:
        return [(int(i), np.float32(d)) for i, d in a]
    ak = pack_keys(np.array([d for _, d in a], np.float32), np.array([i for i, _ in a], np.int64))[None, :]
    bk = pack_keys(np.array([d for _, d in b], np.float32), np.array([i for i, _ in b], np.int64))[None, :]
    dists, ids = unpack_keys(merge_rows(ak, bk)[0])
    return [(int(i), d) for i, d in zip(ids, dists)]


def parallel_merge_sort(items):
    """kernels.py:133-145: sort an (id, dist) list ascending by (dist, id)."""
    items = list(items)
    if len(items) <= 1:
        return [(int(i), np.float32(d)) for i, d in items]
    w = _next_pow2(len(items))
    keys = np.full((1, w), SENTINEL, dtype=np.uint64)
    keys[0, :len(items)] = pack_keys(np.array([d for _, d in items], np.float32),
                                     np.array([i for i, _ in items], np.int64))
    dists, ids = unpack_keys(merge_sort_rows(keys)[0, :len(items)])
    return [(int(i), d) for i, d in zip(ids, dists)]
