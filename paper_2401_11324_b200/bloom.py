"""Per-query Bloom filters (bloom.py:1-163 of the reference).

Hashing is the reference's FNV-1a-64 pair (h1 over the id's four LE bytes,
h2 with 0x5A prepended), slot = h mod entries, bits packed in u64 words.
``BloomFilterBank.filter_and_set`` runs kernel 2 of libbang.so on the GPU
with exact sequential per-row test-and-set semantics.
"""

from __future__ import annotations

import numpy as np

from . import _dev, _lib
from .errors import ParameterError

FNV_OFFSET = np.uint64(0xCBF29CE484222325)
FNV_PRIME = np.uint64(0x100000001B3)
_H2_PREFIX = np.uint64(0x5A)
_BYTE = np.uint64(0xFF)
DEFAULT_ENTRIES = 399_887


def fnv1a_node_hash(node_ids, prefixed: bool = False) -> np.ndarray:
    """bloom.py:26-34 (host; the device computes the same in registers)."""
    ids = np.asarray(node_ids, dtype=np.uint64)
    h = np.full(ids.shape, FNV_OFFSET, dtype=np.uint64)
    with np.errstate(over="ignore"):
        if prefixed:
            h = (h ^ _H2_PREFIX) * FNV_PRIME
        for shift in (np.uint64(0), np.uint64(8), np.uint64(16), np.uint64(24)):
            h = (h ^ ((ids >> shift) & _BYTE)) * FNV_PRIME
    return h


def bit_positions(node_ids, entries: int):
    """bloom.py:37-42: the two filter slots probed for each id."""
    z = np.uint64(entries)
    return fnv1a_node_hash(node_ids) % z, fnv1a_node_hash(node_ids, prefixed=True) % z


class BloomFilterBank:
    """One packed filter per query row, resident on the GPU."""

    def __init__(self, count: int, entries: int = DEFAULT_ENTRIES):
        if entries < 1:
            raise ParameterError("bloom_entries must be positive")
        if entries >= 2 ** 31:
            raise ParameterError("bloom_entries must be < 2^31 on the GPU path")
        self.count = int(count)
        self.entries = int(entries)
        self.words = (self.entries + 63) // 64
        self._bits = _dev.empty((self.count, self.words), np.uint64)
        self._bits.zero_()

    @property
    def bits(self) -> np.ndarray:
        """(count, words) u64 copy of the device filters."""
        return _dev.to_host(self._bits, np.uint64)

    def set_all_rows(self, node_id: int) -> None:
        """bloom.py:87-92: mark one id in every filter (the entry point).
        Through kernel 2: testing-and-setting the id in every row sets both
        of its bits in every row (already-set bits stay set)."""
        self.filter_and_set(np.arange(self.count, dtype=np.int64), np.full(self.count, int(node_id), np.int64))

    def filter_and_set(self, rows, node_ids) -> np.ndarray:
        """bloom.py:124-163: test-and-set every (row, id) probe, equal rows in
        order of appearance; returns the fresh (admitted) mask."""
        rows = np.asarray(rows, dtype=np.int64)
        ids = np.asarray(node_ids)
        if ids.size == 0:
            return np.zeros(0, dtype=bool)
        if rows.size and (rows.min() < 0 or rows.max() >= self.count):
            raise ParameterError("row index out of range")
        order = np.argsort(rows, kind="stable")  # CSR by row, appearance order kept
        offsets = np.zeros(self.count + 1, np.int64)
        np.cumsum(np.bincount(rows, minlength=self.count), out=offsets[1:])
        low32 = (np.asarray(ids, dtype=np.int64)[order] & 0xFFFFFFFF).astype(np.uint32)
        d_off, d_ids = _dev.to_dev(offsets), _dev.to_dev(low32.view(np.int32))
        d_fresh = _dev.empty((ids.size,), np.uint8)
        _lib.check(_lib.lib().bang_bloom_filter_device(
            _lib.ptr(self._bits), self.count, self.entries, _lib.ptr(d_off), _lib.ptr(d_ids),
            _lib.ptr(d_fresh), _lib.stream_ptr(_dev.stream())), "filter_and_set")
        fresh_sorted = _dev.to_host(d_fresh).astype(bool)
        fresh = np.empty(ids.size, dtype=bool)
        fresh[order] = fresh_sorted
        return fresh
