# bang/_gpu.py -- optional B200 backend for the reference GraphSearcher
# (ctypes over libbang.so, include/bang.h).
#
# This is the module a maintainer adds to the reference package
# (/root/reference/pkg/src/bang/) as bang/_gpu.py; INTEGRATION.md shows the
# two-line hook in engine.py that calls it.  It uses only the reference's own
# names (GraphIndex.adjacency/degrees/medoid/node_count, PQCodebook.centroids/
# subspace_sizes/m, CompressedVectors.codes, errors.BangError/ParameterError/
# FileFormatError/TruncatedFileError), so it runs unchanged inside either
# package: tests/test_integration.py loads it under paper_2401_11324_b200 (whose
# classes carry the same names) and checks its outputs against the reference's
# own fixtures.
import ctypes
import os

import numpy as np

from .errors import BangError, FileFormatError, ParameterError, TruncatedFileError

_L = ctypes.CDLL(os.environ.get("BANG_LIBBANG", "libbang.so"))
_P, _I32, _I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
_L.bang_last_error.restype = ctypes.c_char_p
_L.bang_index_create.argtypes = [_I32, _P, _I64, _I32, _P, _P, _I32, _P, _P, _I32, _I32, _P,
                                 _I32, _I32, ctypes.POINTER(_P)]
_L.bang_index_create.restype = _I32
_L.bang_index_destroy.argtypes = [_P]
_L.bang_index_destroy.restype = None
_L.bang_search.argtypes = [_P, _P, _I64, _I32, _I32, _I64, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _I64]
_L.bang_search.restype = _I32
_L.bang_last_visit_logs.argtypes = [_P, _P, _I64]
_L.bang_last_visit_logs.restype = _I32
_L.bang_pq_table.argtypes = [_P, _P, _I64, _P]
_L.bang_pq_table.restype = _I32
_L.bang_read_graph_header.argtypes = [ctypes.c_char_p, _P, _P, _P]
_L.bang_read_graph_header.restype = _I32
_L.bang_read_graph.argtypes = [ctypes.c_char_p, _P, _P, _I64, _I32, _I32]
_L.bang_read_graph.restype = _I32

RERANK, DEBUG_CHECKS, EXACT_DISTANCE = 1, 2, 4
VEC = {np.dtype(np.float32): 0, np.dtype(np.uint8): 1, np.dtype(np.int8): 2}
_ERRORS = {-1: ParameterError, -6: FileFormatError, -7: TruncatedFileError}


def _p(a):
    return None if a is None else a.ctypes.data_as(_P)


def _check(st):
    if st == 0:
        return
    raise _ERRORS.get(st, BangError)(_L.bang_last_error().decode())


class GpuIndex:
    """Replaces IndexHost + the artifacts of GraphSearcher.fit (engine.py:377-407)."""

    def __init__(self, graph, vectors, codebook, codes, device=0, mode="in_memory"):
        vectors = np.ascontiguousarray(vectors)
        self.h = _P()
        self.m = codebook.m if mode != "exact_distance" else 0
        cb = sizes = cv = None
        if self.m:
            cb = np.ascontiguousarray(np.concatenate([np.ravel(c) for c in codebook.centroids]), np.float32)
            sizes = np.asarray(codebook.subspace_sizes, np.int32)
            cv = np.ascontiguousarray(codes.codes, np.uint8)
        self.mode = mode
        _check(_L.bang_index_create(device, _p(cv), graph.node_count, self.m, _p(cb), _p(sizes),
                                    vectors.shape[1], _p(np.ascontiguousarray(graph.adjacency, np.int32)),
                                    _p(np.ascontiguousarray(graph.degrees, np.int32)),
                                    graph.adjacency.shape[1], graph.medoid, _p(vectors), VEC[vectors.dtype],
                                    1 if mode == "pipelined" else 0, ctypes.byref(self.h)))

    def close(self):
        if self.h:
            _L.bang_index_destroy(self.h)
            self.h = _P()

    def __del__(self):
        self.close()

    def pq_table(self, queries):
        """build_pq_dist_table(queries, codebook).table (pq.py:299-319)."""
        q = np.ascontiguousarray(queries, np.float32)
        out = np.empty((q.shape[0], self.m, 256), np.float32)
        _check(_L.bang_pq_table(self.h, _p(q), q.shape[0], _p(out)))
        return out

    def search_batch(self, queries, k, t, bloom_entries, rerank=True, debug_checks=False):
        """Same 7-tuple as _search_batch (engine.py:108-112, 270)."""
        q = np.ascontiguousarray(queries, np.float32)
        nq = q.shape[0]
        ids = np.empty((nq, k), np.int32)
        dists = np.empty((nq, k), np.float32)
        it = np.empty(nq, np.int32)
        conv = np.empty(nq, np.uint8)
        short = np.empty(nq, np.uint8)
        wall = np.empty(nq, np.float64)
        offs = np.empty(nq + 1, np.int64)
        flags = ((RERANK if rerank else 0) | (DEBUG_CHECKS if debug_checks else 0) |
                 (EXACT_DISTANCE if self.mode == "exact_distance" else 0))
        _check(_L.bang_search(self.h, _p(q), nq, k, t, bloom_entries, flags, _p(ids), _p(dists),
                              _p(it), _p(conv), _p(short), _p(wall), _p(offs), None, 0))
        flat = np.empty(int(offs[-1]), np.int32)
        _check(_L.bang_last_visit_logs(self.h, _p(flat), flat.size))
        logs = [flat[offs[i]:offs[i + 1]].astype(np.int64) for i in range(nq)]
        return ids, dists, it, conv.astype(bool), wall, short.astype(bool), logs


def read_graph_arrays(path, threads=0):
    """(adjacency, degrees, medoid, R) of a PGIX file -- the native loader
    behind read_graph (io.py:254-278); wrap in GraphIndex(...)."""
    n, R, med = _I64(), _I32(), _I32()
    bpath = os.fsencode(path)
    _check(_L.bang_read_graph_header(bpath, ctypes.byref(n), ctypes.byref(R), ctypes.byref(med)))
    adj = np.empty((n.value, R.value), np.int32)
    deg = np.empty(n.value, np.int32)
    _check(_L.bang_read_graph(bpath, _p(adj), _p(deg), n.value, R.value, threads))
    return adj, deg, med.value, R.value
