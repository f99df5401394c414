"""Product-quantization containers and the on-device table/ADC (pq.py).

Containers mirror the reference (pq.py:27-124).  ``build_pq_dist_table``
runs kernel 1 and ``asymmetric_distance(s)`` kernel 3 of libbang.so.
Codebook training is offline index construction (out of the hot path); the
GPU trainer used by the benchmarks lives in ``tools/pq_train.py``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .errors import ParameterError
from .validation import as_float32_rows, check_matrix, check_positive

CENTROIDS_PER_SUBSPACE = 256


def subspace_split(dim: int, m: int) -> list[int]:
    """pq.py:27-34: the first dim % m subspaces get the extra dimension."""
    check_positive("m", m)
    check_positive("dim", dim)
    if m > dim:
        raise ParameterError(f"m={m} exceeds dim={dim}")
    base, extra = divmod(dim, m)
    return [base + 1] * extra + [base] * (m - extra)


@dataclass
class PQCodebook:
    dim: int
    subspace_sizes: list
    centroids: list  # m arrays (256, subspace_sizes[s]) f32

    def __post_init__(self):
        if sum(self.subspace_sizes) != self.dim:
            raise ParameterError(f"subspace sizes sum to {sum(self.subspace_sizes)}, expected {self.dim}")
        if len(self.centroids) != len(self.subspace_sizes):
            raise ParameterError("one centroid table per subspace required")
        for s, (table, size) in enumerate(zip(self.centroids, self.subspace_sizes)):
            if np.shape(table) != (CENTROIDS_PER_SUBSPACE, size):
                raise ParameterError(f"subspace {s}: centroid table shape {np.shape(table)}, "
                                     f"expected ({CENTROIDS_PER_SUBSPACE}, {size})")
            self.centroids[s] = np.ascontiguousarray(table, dtype=np.float32)

    @property
    def m(self) -> int:
        return len(self.subspace_sizes)

    def offsets(self) -> list:
        out, pos = [], 0
        for size in self.subspace_sizes:
            out.append(pos)
            pos += size
        return out

    def concatenated(self) -> np.ndarray:
        """The device layout: subspace tables back to back, (256*dim,) f32."""
        return np.ascontiguousarray(np.concatenate([c.ravel() for c in self.centroids]), dtype=np.float32)

    def __eq__(self, other) -> bool:
        if not isinstance(other, PQCodebook):
            return NotImplemented
        return (self.dim == other.dim and list(self.subspace_sizes) == list(other.subspace_sizes)
                and all(np.array_equal(a, b) for a, b in zip(self.centroids, other.centroids)))


@dataclass
class CompressedVectors:
    codes: np.ndarray  # (count, m) uint8

    def __post_init__(self):
        self.codes = np.ascontiguousarray(self.codes, dtype=np.uint8)
        if self.codes.ndim != 2:
            raise ParameterError("codes must be a (count, m) matrix")

    @property
    def count(self) -> int:
        return self.codes.shape[0]

    @property
    def m(self) -> int:
        return self.codes.shape[1]


@dataclass
class PQDistTable:
    table: np.ndarray  # (rho, m, 256) float32

    def __post_init__(self):
        self.table = np.ascontiguousarray(self.table, dtype=np.float32)
        if self.table.ndim != 3 or self.table.shape[2] != CENTROIDS_PER_SUBSPACE:
            raise ParameterError("table must have shape (rho, m, 256)")

    @property
    def rho(self) -> int:
        return self.table.shape[0]

    @property
    def m(self) -> int:
        return self.table.shape[1]

    @property
    def flat(self) -> np.ndarray:
        return self.table.reshape(-1)


def build_pq_dist_table(queries, codebook: PQCodebook, threads=None) -> PQDistTable:
    """pq.py:299-319 on the GPU (kernel 1); ``threads`` is accepted for API
    compatibility -- the result is bit-identical for any value."""
    data = queries.data if hasattr(queries, "data") else queries
    q = as_float32_rows(check_matrix(data, "queries"))
    if q.shape[1] != codebook.dim:
        raise ParameterError(f"query dim {q.shape[1]} != codebook dim {codebook.dim}")
    rho = q.shape[0]
    if rho == 0:
        return PQDistTable(np.empty((0, codebook.m, 256), np.float32))
    dq, dcb = _dev.to_dev(q), _dev.to_dev(codebook.concatenated())
    out = _dev.empty((rho, codebook.m, 256), np.float32)
    sizes = np.ascontiguousarray(codebook.subspace_sizes, dtype=np.int32)
    _lib.check(_lib.lib().bang_pq_table_device(_lib.ptr(dcb), _lib.ptr(sizes), codebook.m, codebook.dim,
                                               _lib.ptr(dq), rho, _lib.ptr(out),
                                               _lib.stream_ptr(_dev.stream())), "build_pq_dist_table")
    return PQDistTable(_dev.to_host(out))


def _adc_pairs(table: PQDistTable, codes: np.ndarray, qrows: np.ndarray, ids: np.ndarray) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    if ids.size == 0:
        return np.zeros(0, np.float32)
    dt, dc = _dev.to_dev(table.table), _dev.to_dev(codes)
    dq = _dev.to_dev(np.ascontiguousarray(qrows, dtype=np.int64))
    di = _dev.to_dev(np.ascontiguousarray(ids, dtype=np.int64).astype(np.uint32).view(np.int32))
    out = _dev.empty((ids.size,), np.float32)
    _lib.check(_lib.lib().bang_adc_device(_lib.ptr(dt), table.m, _lib.ptr(dc), _lib.ptr(dq), _lib.ptr(di),
                                          ids.size, _lib.ptr(out), None, _lib.stream_ptr(_dev.stream())),
               "asymmetric_distances")
    return _dev.to_host(out)


def asymmetric_distance(code, query_index: int, table: PQDistTable) -> np.float32:
    """pq.py:322-333: sum of table entries over s = 0..m-1 in f32 (kernel 3)."""
    if not 0 <= query_index < table.rho:
        raise ParameterError(f"query index {query_index} out of range")
    code = np.asarray(code)
    if code.shape != (table.m,):
        raise ParameterError(f"code must have {table.m} entries, got {code.shape}")
    return np.float32(_adc_pairs(table, code[None, :], np.array([query_index]), np.array([0]))[0])


def asymmetric_distances(codes: CompressedVectors, node_ids, query_index: int,
                         table: PQDistTable) -> np.ndarray:
    """pq.py:336-345 (kernel 3)."""
    ids = np.asarray(node_ids, dtype=np.int64)
    return _adc_pairs(table, codes.codes, np.full(ids.size, query_index, np.int64), ids)


def compute_neighbour_distances(codes: CompressedVectors, node_ids, query_index: int,
                                table: PQDistTable):
    """pq.py:348-354."""
    ids = np.asarray(node_ids, dtype=np.int64)
    dists = asymmetric_distances(codes, ids, query_index, table)
    return [(int(i), d) for i, d in zip(ids, dists)]
