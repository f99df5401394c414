"""ctypes wrapper over liboracle.so -- the CPU restatement of the reference.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg; never by the product
package ``paper_2401_11324_b200``.  Each function names the reference
function it restates (paths under /root/reference/pkg/src/bang/).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

SENTINEL = np.uint64(0xFFFFFFFFFFFFFFFF)
DTYPE_CODES = {np.dtype(np.float32): 0, np.dtype(np.uint8): 1, np.dtype(np.int8): 2}

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_U64 = ctypes.c_uint64


def build() -> str:
    """Compile liboracle.so with the committed Makefile (idempotent)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.bo_pq_table.argtypes = [_P, _I64, _I32, _P, _P, _I32, _P]
        L.bo_fnv1a.argtypes = [_U64, _I32]
        L.bo_fnv1a.restype = _U64
        L.bo_bit_positions.argtypes = [_P, _I64, _U64, _P, _P]
        L.bo_bloom_filter_and_set.argtypes = [_P, _I64, _U64, _P, _P, _I64, _P]
        L.bo_adc.argtypes = [_P, _I32, _P, _P, _P, _I64, _P]
        L.bo_pack.argtypes = [ctypes.c_float, ctypes.c_uint32]
        L.bo_pack.restype = _U64
        L.bo_sort_rows.argtypes = [_P, _I64, _I32]
        L.bo_merge_rows.argtypes = [_P, _P, _I64, _I32, _P, _I32, _P, _P]
        L.bo_exact_sq_dist.argtypes = [_P, _I32, _P, _I32]
        L.bo_exact_sq_dist.restype = ctypes.c_float
        L.bo_rerank.argtypes = [_P, _I32, _P, _I32, _I32, _P, _I32, _P, _P]
        L.bo_rerank.restype = _I32
        L.bo_search.argtypes = [_P, _I64, _I32, _P, _P, _I32, _P, _P, _P, _P, _I64,
                                _I32, _I32, _P, _I32, _I32, _I32, _U64, _I32, _I32,
                                _I32, _P, _P, _P, _P, _P, _P, _I64]
        L.bo_search.restype = _I64
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _concat_centroids(centroids):
    return np.ascontiguousarray(np.concatenate([np.ascontiguousarray(c, np.float32).ravel()
                                                for c in centroids]))


def pq_table(queries, centroids, sub_sizes):
    """pq.py:299-319 build_pq_dist_table -> (nq, m, 256) f32."""
    q = np.ascontiguousarray(queries, dtype=np.float32)
    sizes = np.ascontiguousarray(sub_sizes, dtype=np.int32)
    cb = _concat_centroids(centroids)
    out = np.empty((q.shape[0], sizes.size, 256), np.float32)
    lib().bo_pq_table(_ptr(q), q.shape[0], q.shape[1], _ptr(cb), _ptr(sizes), sizes.size, _ptr(out))
    return out


def bit_positions(ids, entries):
    """bloom.py:37-42."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    p1 = np.empty(ids.size, np.uint64)
    p2 = np.empty(ids.size, np.uint64)
    lib().bo_bit_positions(_ptr(ids), ids.size, int(entries), _ptr(p1), _ptr(p2))
    return p1, p2


def bloom_filter_and_set(bits, entries, rows, ids):
    """bloom.py:124-163 on a (count, words) u64 bank, updated in place."""
    assert bits.dtype == np.uint64 and bits.flags.c_contiguous
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    fresh = np.zeros(ids.size, np.uint8)
    lib().bo_bloom_filter_and_set(_ptr(bits), bits.shape[0], int(entries), _ptr(rows),
                                  _ptr(ids), ids.size, _ptr(fresh))
    return fresh.astype(bool)


def adc(table, codes, qrows, ids):
    """engine.py:99-105 _pq_point_dists."""
    table = np.ascontiguousarray(table, dtype=np.float32)
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    qrows = np.ascontiguousarray(qrows, dtype=np.int64)
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    out = np.empty(ids.size, np.float32)
    lib().bo_adc(_ptr(table), table.shape[1], _ptr(codes), _ptr(qrows), _ptr(ids), ids.size, _ptr(out))
    return out


def pack_keys(dists, ids):
    """kernels.py:25-29."""
    d = np.ascontiguousarray(dists, dtype=np.float32)
    return (d.view(np.uint32).astype(np.uint64) << np.uint64(32)) | np.asarray(ids, np.uint64)


def sort_rows(keys):
    """kernels.py:94-109 merge_sort_rows."""
    k = np.array(keys, dtype=np.uint64, order="C", copy=True)
    lib().bo_sort_rows(_ptr(k), k.shape[0], k.shape[1])
    return k


def merge_rows(a, b, a_payload=None):
    """kernels.py:68-87."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    n, wa = a.shape
    wb = b.shape[1]
    out = np.empty((n, wa + wb), np.uint64)
    pay = None if a_payload is None else np.ascontiguousarray(a_payload, dtype=np.uint8)
    out_pay = np.empty((n, wa + wb), np.uint8)
    lib().bo_merge_rows(_ptr(a), _ptr(pay), n, wa, _ptr(b), wb, _ptr(out), _ptr(out_pay))
    if a_payload is None:
        return out
    return out, out_pay.astype(bool)


def exact_sq_dists(points, queries):
    """engine.py:48-51 (row-paired)."""
    p = np.ascontiguousarray(points)
    q = np.ascontiguousarray(queries, dtype=np.float32)
    code = DTYPE_CODES[p.dtype]
    out = np.empty(p.shape[0], np.float32)
    for i in range(p.shape[0]):
        out[i] = lib().bo_exact_sq_dist(_ptr(p[i]), code, _ptr(q[i]), p.shape[1])
    return out


def search(queries, *, centroids, sub_sizes, codes, adjacency, degrees, medoid,
           vectors, k, t, bloom_entries, rerank=True, mode="pq", table=None,
           threads=1, log_cap=None):
    """engine.py:108-270 _search_batch (+ table build) over a batch.

    Returns dict(ids, dists, iterations, converged, short, visit_logs).
    """
    q = np.ascontiguousarray(queries, dtype=np.float32)
    nq, dim = q.shape
    vec = np.ascontiguousarray(vectors)
    adjacency = np.ascontiguousarray(adjacency, dtype=np.int32)
    degrees = np.ascontiguousarray(degrees, dtype=np.int32)
    n, R = adjacency.shape
    mode_code = 0 if mode == "pq" else 1
    if mode_code == 0:
        cb = _concat_centroids(centroids)
        sizes = np.ascontiguousarray(sub_sizes, dtype=np.int32)
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        m = sizes.size
    else:
        cb = sizes = codes = None
        m = 0
    tab = None if table is None else np.ascontiguousarray(table, dtype=np.float32)
    cap = int(log_cap) if log_cap else max(4 * t, 64)
    while True:
        ids = np.empty((nq, k), np.int32)
        dists = np.empty((nq, k), np.float32)
        iters = np.zeros(nq, np.int32)
        conv = np.zeros(nq, np.uint8)
        short = np.zeros(nq, np.uint8)
        logs = np.zeros((nq, cap), np.int32)
        need = lib().bo_search(_ptr(q), nq, dim, _ptr(cb), _ptr(sizes), m, _ptr(tab),
                               _ptr(codes), _ptr(adjacency), _ptr(degrees), n, R,
                               int(medoid), _ptr(vec), DTYPE_CODES[vec.dtype], k, t,
                               int(bloom_entries), int(bool(rerank)), mode_code,
                               int(threads), _ptr(ids), _ptr(dists), _ptr(iters),
                               _ptr(conv), _ptr(short), _ptr(logs), cap)
        if need == 0:
            break
        cap = int(need)
    return dict(ids=ids, dists=dists, iterations=iters, converged=conv.astype(bool),
                short=short.astype(bool),
                visit_logs=[logs[i, :iters[i]].astype(np.int64) for i in range(nq)])
