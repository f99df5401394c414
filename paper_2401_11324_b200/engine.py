"""Drop-in batched search engine: the reference's GraphSearcher API
(engine.py:335-460) over the B200 kernels of libbang.so.

``fit`` uploads the index once (codes + codebook + graph + re-rank vectors
to HBM, or graph/vectors pinned+mapped in host memory for
``mode="pipelined"``); ``search`` runs each ``batch_size`` chunk through the
fused persistent search kernel (bang_search) and returns the reference's
``SearchResult``.  Results equal the reference's bit for bit: visit logs,
iterations, ids, distances, short flags (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import ctypes
import time
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .bloom import DEFAULT_ENTRIES
from .errors import BangError, ParameterError
from .graph import GraphIndex
from .kernels import SENTINEL, merge_sort_rows, pack_keys, unpack_keys, _next_pow2
from .pq import CompressedVectors, PQCodebook
from .validation import as_engine_rows, as_float32_rows, check_matrix, check_positive

try:  # the reference is a scikit-learn estimator; keep get_params/clone working
    from sklearn.base import BaseEstimator
except ImportError:  # pragma: no cover
    class BaseEstimator:  # minimal stand-in with the same params protocol
        def get_params(self, deep=True):
            import inspect
            names = [p for p in inspect.signature(self.__init__).parameters if p != "self"]
            return {n: getattr(self, n) for n in names}

MODES = ("pipelined", "in_memory", "exact_distance")
_VEC_CODE = {np.dtype(np.float32): _lib.VEC_F32, np.dtype(np.uint8): _lib.VEC_U8,
             np.dtype(np.int8): _lib.VEC_I8}


class VisitLogs(Sequence):
    """Per-query visit logs as a read-only list of int64 arrays, backed by one
    CSR buffer (offsets + flat ids) so a 10K-query batch costs no Python
    loop; ``logs[i]`` is query i's expanded ids in visit order."""

    def __init__(self, parts):
        self._offs = []
        self._flat = []
        self._base = [0]
        for offs, flat in parts:
            self._offs.append(np.asarray(offs, np.int64))
            # ids stay in the device's int32 until a log is read: logs[i]
            # returns int64 like the reference, without widening 10^6+ ids
            # per batch up front
            self._flat.append(np.asarray(flat))
            self._base.append(self._base[-1] + len(offs) - 1)

    def __len__(self):
        return self._base[-1]

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        n = len(self)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError("visit log index out of range")
        p = int(np.searchsorted(self._base, i, side="right")) - 1
        j = i - self._base[p]
        offs = self._offs[p]
        return self._flat[p][offs[j]:offs[j + 1]].astype(np.int64)

    def __eq__(self, other):
        return len(self) == len(other) and all(np.array_equal(a, b) for a, b in zip(self, other))

    def csr(self):
        """(offsets (n+1,) int64, ids int64): all logs as one CSR pair."""
        if len(self._offs) == 1:
            return self._offs[0], self._flat[0].astype(np.int64, copy=False)
        offs, flats, base = [np.zeros(1, np.int64)], [], 0
        for o, f in zip(self._offs, self._flat):
            offs.append(o[1:] - o[0] + base)
            flats.append(f[o[0]:o[-1]])
            base += int(o[-1] - o[0])
        return np.concatenate(offs), (np.concatenate(flats).astype(np.int64, copy=False) if flats
                                      else np.zeros(0, np.int64))

    @classmethod
    def concat(cls, logs_list) -> "VisitLogs":
        """Logs of several batches/shards, in order (plain lists accepted)."""
        out = cls([])
        for logs in logs_list:
            if isinstance(logs, VisitLogs):
                for offs, flat in zip(logs._offs, logs._flat):
                    out._offs.append(offs)
                    out._flat.append(flat)
                    out._base.append(out._base[-1] + len(offs) - 1)
            else:
                arrs = [np.asarray(a, np.int64) for a in logs]
                offs = np.zeros(len(arrs) + 1, np.int64)
                if arrs:
                    offs[1:] = np.cumsum([a.size for a in arrs])
                flat = np.concatenate(arrs) if arrs else np.zeros(0, np.int64)
                out._offs.append(offs)
                out._flat.append(flat)
                out._base.append(out._base[-1] + len(arrs))
        return out


@dataclass
class SearchResult:
    """Per-query outputs of a batched search (engine.py:85-96)."""

    ids: np.ndarray          # (nq, k) int32, -1 padding when short
    dists: np.ndarray        # (nq, k) float32, +inf padding
    iterations: np.ndarray   # (nq,) int32
    converged: np.ndarray    # (nq,) bool
    wall_times: np.ndarray   # (nq,) float64, seconds from batch start (device clock)
    elapsed: float           # total search seconds over all batches
    short: np.ndarray        # (nq,) bool
    visit_logs: list         # per query, expanded node ids in visit order (int64)


class IndexHost:
    """The host domain of the reference (engine.py:54-72): graph + vectors."""

    def __init__(self, graph: GraphIndex, vectors: np.ndarray):
        vectors = check_matrix(vectors, "vectors")
        if vectors.shape[0] != graph.node_count:
            raise ParameterError("vector count does not match the graph")
        self.graph = graph
        self.vectors = vectors

    def fetch(self, node_ids):
        ids = np.asarray(node_ids, dtype=np.int64)
        return (self.graph.adjacency[ids], self.graph.degrees[ids],
                as_float32_rows(self.vectors[ids]))


class DeviceIndex:
    """Owner of one ``bang_index`` handle (one GPU)."""

    def __init__(self, graph: GraphIndex, vectors: np.ndarray, codebook: PQCodebook | None,
                 codes: CompressedVectors | None, placement: int, device: int | None = None):
        L = _lib.lib()
        self.device = _dev.device_index() if device is None else int(device)
        vec = as_engine_rows(vectors)
        self.dim = vec.shape[1]
        self.n = graph.node_count
        if codebook is not None:
            cb = codebook.concatenated()
            sizes = np.ascontiguousarray(codebook.subspace_sizes, dtype=np.int32)
            cds = np.ascontiguousarray(codes.codes, dtype=np.uint8)
            m = codebook.m
        else:
            cb = sizes = cds = None
            m = 0
        handle = ctypes.c_void_p()
        adj = np.ascontiguousarray(graph.adjacency, dtype=np.int32)
        deg = np.ascontiguousarray(graph.degrees, dtype=np.int32)
        st = L.bang_index_create(self.device, _lib.ptr(cds), self.n, m, _lib.ptr(cb), _lib.ptr(sizes),
                                 self.dim, _lib.ptr(adj), _lib.ptr(deg), adj.shape[1], graph.medoid,
                                 _lib.ptr(vec), _VEC_CODE[vec.dtype], placement, ctypes.byref(handle))
        _lib.check(st, "bang_index_create")
        self.handle = handle
        self.m = m

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            _lib.lib().bang_index_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def search(self, queries: np.ndarray, k: int, t: int, bloom_entries: int, flags: int):
        q = np.ascontiguousarray(queries, dtype=np.float32)
        nq = q.shape[0]
        # the large device->host results land in page-locked memory
        ids = _dev.pinned_empty((nq, k), np.int32)
        dists = _dev.pinned_empty((nq, k), np.float32)
        iters = np.empty(nq, np.int32)
        conv = np.empty(nq, np.uint8)
        short = np.empty(nq, np.uint8)
        wall = np.empty(nq, np.float64)
        offs = np.empty(nq + 1, np.int64)
        # a page-locked log buffer for the worst case (nq x the default device
        # log capacity, bang.h) lets bang_search compact the visit logs
        # straight into it and read everything back in one batch
        flat = _dev.pinned_empty(nq * max(1024, 4 * t), np.int32)
        L = _lib.lib()
        st = L.bang_search(self.handle, _lib.ptr(q), nq, k, t, int(bloom_entries), flags, _lib.ptr(ids),
                           _lib.ptr(dists), _lib.ptr(iters), _lib.ptr(conv), _lib.ptr(short),
                           _lib.ptr(wall), _lib.ptr(offs), _lib.ptr(flat), flat.size)
        if st == _lib.BANG_E_CAPACITY:  # longer logs (re-runs): the two-call protocol
            flat = _dev.pinned_empty(int(offs[-1]), np.int32)
            st = L.bang_last_visit_logs(self.handle, _lib.ptr(flat), flat.size)
        _lib.check(st, "bang_search")
        return ids, dists, iters, conv.astype(bool), short.astype(bool), wall, offs, flat[:int(offs[-1])]

    def stats(self) -> dict:
        s = _lib.SearchStats()
        _lib.check(_lib.lib().bang_last_search_stats(self.handle, ctypes.byref(s)))
        return s.as_dict()

    def options(self) -> dict:
        o = _lib.Options()
        _lib.check(_lib.lib().bang_index_get_options(self.handle, ctypes.byref(o)), "bang_index_get_options")
        return o.as_dict()

    def set_options(self, kernel: str = "auto", **tuning) -> None:
        """bang_index_set_options: kernel in _lib.KERNEL_CHOICES plus the
        bang_options tuning fields (row_prefetch, bloom_clear, l2_persist,
        profile); unnamed fields keep their defaults."""
        if kernel not in _lib.KERNEL_CHOICES:
            raise ParameterError(f"unknown kernel {kernel!r}; expected one of {sorted(_lib.KERNEL_CHOICES)}")
        o = _lib.Options()
        L = _lib.lib()
        L.bang_options_default(ctypes.byref(o))
        o.kernel = _lib.KERNEL_CHOICES[kernel]
        for name, value in tuning.items():
            if name not in o.as_dict() or name == "kernel":
                raise ParameterError(f"unknown search option {name!r}")
            setattr(o, name, int(value))
        _lib.check(L.bang_index_set_options(self.handle, ctypes.byref(o)), "bang_index_set_options")

    def pq_table(self, queries: np.ndarray) -> np.ndarray:
        """bang_pq_table: kernel 1 on host buffers (pq.py:299-319)."""
        q = np.ascontiguousarray(queries, dtype=np.float32)
        out = np.empty((q.shape[0], self.m, 256), np.float32)
        _lib.check(_lib.lib().bang_pq_table(self.handle, _lib.ptr(q), q.shape[0], _lib.ptr(out)), "bang_pq_table")
        return out


def exact_sq_dists(points, queries) -> np.ndarray:
    """engine.py:48-51 on the GPU: row-paired squared L2, f64 sums -> f32."""
    p = as_engine_rows(check_matrix(points, "points"))
    q = as_float32_rows(np.ascontiguousarray(np.broadcast_to(queries, p.shape), dtype=np.float32))
    if p.shape[0] == 0:
        return np.zeros(0, np.float32)
    dp, dq = _dev.to_dev(p), _dev.to_dev(q)
    out = _dev.empty((p.shape[0],), np.float32)
    _lib.check(_lib.lib().bang_exact_sq_dists_device(_lib.ptr(dp), _VEC_CODE[p.dtype], p.shape[1],
                                                     _lib.ptr(dq), p.shape[0], _lib.ptr(out),
                                                     _lib.stream_ptr(_dev.stream())), "exact_sq_dists")
    return _dev.to_host(out)


def rerank(candidate_ids, candidate_vectors, query, k: int):
    """engine.py:273-292: exact-distance ordering of one query's candidates."""
    ids = np.asarray(candidate_ids, dtype=np.int64)
    vecs = check_matrix(candidate_vectors, "candidate_vectors")
    q = as_float32_rows(np.asarray(query, dtype=np.float32).reshape(1, -1))[0]
    if ids.size != vecs.shape[0]:
        raise ParameterError("one vector per candidate id required")
    if ids.size == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.float32), k > 0
    dists = exact_sq_dists(vecs, np.broadcast_to(q, (vecs.shape[0], q.size)))
    keys = np.full((1, _next_pow2(ids.size)), SENTINEL, dtype=np.uint64)
    keys[0, :ids.size] = pack_keys(dists, ids)
    ordered = merge_sort_rows(keys)[0, :min(k, ids.size)]
    d_out, i_out = unpack_keys(ordered)
    return i_out, d_out, ids.size < k


class GraphSearcher(BaseEstimator):
    """Batched approximate k-NN search over a graph index (engine.py:335-460).

    Same constructor parameters, defaults, checks and outputs as the
    reference.  ``mode`` picks where the graph lives: "in_memory" (HBM),
    "pipelined" (pinned, mapped host memory read over PCIe with the next
    hop prefetched) or "exact_distance" (exact f64->f32 scoring, no codes,
    no re-rank).  ``threads`` is accepted and ignored (the GPU result does
    not depend on it, as the reference's does not).
    """

    def __init__(self, k: int = 10, t: int = 152, mode: str = "pipelined",
                 bloom_entries: int = DEFAULT_ENTRIES, batch_size: int = 10_000,
                 rerank: bool = True, degree_bound: int = 64,
                 build_worklist: int = 200, sigma: float = 1.2, m: int = 74,
                 pq_iters: int = 25, seed: int = 0, threads: int | None = None,
                 debug_checks: bool = False):
        self.k = k
        self.t = t
        self.mode = mode
        self.bloom_entries = bloom_entries
        self.batch_size = batch_size
        self.rerank = rerank
        self.degree_bound = degree_bound
        self.build_worklist = build_worklist
        self.sigma = sigma
        self.m = m
        self.pq_iters = pq_iters
        self.seed = seed
        self.threads = threads
        self.debug_checks = debug_checks

    def _check_params(self):
        """engine.py:368-375."""
        check_positive("k", self.k)
        if self.t < self.k:
            raise ParameterError(f"t={self.t} must be >= k={self.k}")
        if self.mode not in MODES:
            raise ParameterError(f"mode must be one of {MODES}, got {self.mode!r}")
        check_positive("bloom_entries", self.bloom_entries)
        check_positive("batch_size", self.batch_size)

    def fit(self, X, y=None, graph: GraphIndex | None = None, codebook: PQCodebook | None = None,
            codes: CompressedVectors | None = None) -> "GraphSearcher":
        """engine.py:377-407: attach (or build) the artifacts and upload them."""
        self._check_params()
        data = getattr(X, "data", X)
        base = as_engine_rows(check_matrix(data, "X"))
        if graph is None:
            from .tools.graph_build import build_graph
            graph = build_graph(base, degree_bound=self.degree_bound, build_worklist=self.build_worklist,
                                sigma=self.sigma, seed=self.seed)
        if graph.node_count != base.shape[0]:
            raise ParameterError("graph node count does not match the base set")
        if self.mode != "exact_distance":
            if codebook is None:
                from .tools.pq_train import train_codebook
                codebook = train_codebook(base, m=self.m, iters=self.pq_iters, seed=self.seed)
            if codebook.dim != base.shape[1]:
                raise ParameterError("codebook dimension does not match the base set")
            if codes is None:
                from .tools.pq_train import encode
                codes = encode(base, codebook)
            if codes.count != base.shape[0] or codes.m != codebook.m:
                raise ParameterError("compressed vectors do not match base/codebook")
        else:
            codebook, codes = None, None
        placement = _lib.GRAPH_HOST_MAPPED if self.mode == "pipelined" else _lib.GRAPH_HBM
        # ``device`` (not a constructor parameter): the GPU this replica uses
        # (sharding.ShardedSearcher sets one per replica); default BANG_DEVICE/LOCAL_RANK.
        # The new index is created before the old one is released, so a failed
        # re-fit (e.g. out of memory) leaves the previous index usable.
        new_index = DeviceIndex(graph, base, codebook, codes, placement, device=getattr(self, "device", None))
        opts = getattr(self, "_kernel_options", None)
        try:
            if opts is not None:
                new_index.set_options(**opts)
            if self.mode == "in_memory":
                # the split kernel's per-(index, Bloom size) row flags now,
                # not on the first search (bang_index_prepare)
                _lib.check(_lib.lib().bang_index_prepare(new_index.handle, int(self.bloom_entries)),
                           "bang_index_prepare")
        except Exception:
            new_index.close()
            raise
        old = getattr(self, "index_", None)
        self.index_ = new_index
        if old is not None:
            old.close()
        self.host_ = IndexHost(graph, base)
        self.graph_ = graph
        self.codebook_ = codebook
        self.codes_ = codes
        self.engine_vectors_ = base if self.mode != "pipelined" else None
        return self

    _ADC_FLAGS = {"auto": 0, "smem-table": _lib.TABLE_SMEM, "codebook": _lib.CODEBOOK_SMEM,
                  "hbm-table": _lib.TABLE_GLOBAL}

    def set_adc_variant(self, name: str) -> "GraphSearcher":
        """Pick the ADC data flow (results are identical for all of them):
        "auto", "smem-table" (per-query table in shared memory, the paper's
        layout), "codebook" (entries recomputed from a CTA-shared codebook) or
        "hbm-table" (kernel 1 writes the table to HBM)."""
        if name not in self._ADC_FLAGS:
            raise ParameterError(f"unknown ADC variant {name!r}")
        self._adc_variant = name
        return self

    def set_kernel(self, kernel: str = "auto", **tuning) -> "GraphSearcher":
        """Pick the search kernel ("auto", "warp", "cta", "split") and its tuning
        (bang_options in include/bang.h).  Results are identical for every
        choice; this only moves work between warps and memory levels."""
        self._kernel_options = dict(kernel=kernel, **tuning)
        if getattr(self, "index_", None) is not None:
            self.index_.set_options(**self._kernel_options)
        return self

    def _flags(self) -> int:
        flags = self._ADC_FLAGS[getattr(self, "_adc_variant", "auto")]
        if self.rerank:
            flags |= _lib.RERANK
        if self.debug_checks:
            flags |= _lib.DEBUG_CHECKS
        if self.mode == "exact_distance":
            flags |= _lib.EXACT_DISTANCE
        return flags

    def search(self, queries, k: int | None = None) -> SearchResult:
        """engine.py:409-452; deterministic for fixed inputs and params."""
        if not hasattr(self, "host_"):
            raise ParameterError("GraphSearcher is not fitted")
        k = self.k if k is None else int(k)
        if k < 1 or k > self.t:
            raise ParameterError(f"k={k} must be in [1, t={self.t}]")
        data = getattr(queries, "data", queries)
        # finiteness of f32 queries: checked by bang_search on the device
        # (same message); other float types on the host before the cast (the
        # device then also rejects values the f32 cast turned into inf)
        arr = np.asarray(data)
        q = as_float32_rows(check_matrix(arr, "queries", finite=arr.dtype != np.float32))
        nq = q.shape[0]
        if nq == 0:
            return SearchResult(np.zeros((0, k), np.int32), np.zeros((0, k), np.float32),
                                np.zeros(0, np.int32), np.zeros(0, bool), np.zeros(0, np.float64), 0.0,
                                np.zeros(0, bool), [])
        if q.shape[1] != self.host_.vectors.shape[1]:
            raise ParameterError("query dimension does not match the base set")
        parts = []
        elapsed = 0.0
        flags = self._flags()
        for lo in range(0, nq, self.batch_size):
            hi = min(nq, lo + self.batch_size)
            t0 = time.perf_counter()
            parts.append(self.index_.search(q[lo:hi], k, self.t, self.bloom_entries, flags))
            elapsed += time.perf_counter() - t0
        logs = VisitLogs([(p[6], p[7]) for p in parts])
        if len(parts) == 1:  # one batch: the arrays as returned (no copies)
            p = parts[0]
            return SearchResult(ids=p[0], dists=p[1], iterations=p[2], converged=p[3], wall_times=p[5],
                                elapsed=elapsed, short=p[4], visit_logs=logs)
        return SearchResult(
            ids=np.concatenate([p[0] for p in parts]),
            dists=np.concatenate([p[1] for p in parts]),
            iterations=np.concatenate([p[2] for p in parts]),
            converged=np.concatenate([p[3] for p in parts]),
            wall_times=np.concatenate([p[5] for p in parts]),
            elapsed=elapsed,
            short=np.concatenate([p[4] for p in parts]),
            visit_logs=logs)

    def kneighbors(self, queries, n_neighbors: int | None = None, return_distance: bool = True):
        """scikit-learn style accessor over :meth:`search` (engine.py:454-460)."""
        result = self.search(queries, k=n_neighbors)
        if return_distance:
            return result.dists, result.ids
        return result.ids

    def last_stats(self) -> dict:
        """Counters of the last batch (iterations, probes, ADC pairs, kernel ms)."""
        return self.index_.stats()
