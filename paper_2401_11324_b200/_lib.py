"""ctypes binding of libbang.so (the C-ABI declared in include/bang.h).

There is no fallback: if the shared library is missing or no CUDA device is
visible, every entry point raises :class:`BangError` loudly.  The library is
built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
"""

from __future__ import annotations

import ctypes
import os

from .errors import BangError, FileFormatError, ParameterError, TruncatedFileError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbang.so")

BANG_OK = 0
BANG_E_PARAM = -1
BANG_E_CUDA = -2
BANG_E_OOM = -3
BANG_E_CAPACITY = -4
BANG_E_STATE = -5
BANG_E_FORMAT = -6
BANG_E_TRUNCATED = -7

VEC_F32, VEC_U8, VEC_I8 = 0, 1, 2
GRAPH_HBM, GRAPH_HOST_MAPPED = 0, 1

RERANK = 1
DEBUG_CHECKS = 2
EXACT_DISTANCE = 4
TABLE_GLOBAL = 8
TABLE_SMEM = 16
CODEBOOK_SMEM = 32
PROFILE_PHASES = 64
ADC_VARIANTS = {0: "smem-codebook", 1: "hbm-table", 2: "exact", 3: "smem-table"}
# bang_search_stats.kernel -> kernel name
KERNELS = {0: "search_kernel", 2: "search_cta_kernel", 8: "search_split_kernel"}
# bang_options.kernel
KERNEL_CHOICES = {"auto": 0, "warp": 1, "cta": 2, "split": 4}

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32


class Options(ctypes.Structure):
    """bang_options (include/bang.h): per-index kernel choice and tuning."""
    _fields_ = [
        ("kernel", ctypes.c_int32), ("row_prefetch", ctypes.c_int32), ("bloom_clear", ctypes.c_int32),
        ("l2_persist", ctypes.c_int32), ("profile", ctypes.c_int32), ("bloom_direct", ctypes.c_int32),
        ("head_row", ctypes.c_int32), ("reserved", ctypes.c_int32 * 9),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_ if name != "reserved"}


class SearchStats(ctypes.Structure):
    _fields_ = [
        ("queries", ctypes.c_int64), ("iterations", ctypes.c_int64),
        ("probes", ctypes.c_int64), ("fresh", ctypes.c_int64),
        ("rerank_cands", ctypes.c_int64), ("retries", ctypes.c_int64),
        ("slots", ctypes.c_int32), ("warps_per_cta", ctypes.c_int32),
        ("ctas", ctypes.c_int32), ("adc_variant", ctypes.c_int32),
        ("kernel_ms", ctypes.c_float), ("table_ms", ctypes.c_float),
        ("algorithmic_bytes", ctypes.c_int64), ("adc_bytes", ctypes.c_int64),
        ("phase_cycles", ctypes.c_int64 * 8),
        ("kernel", ctypes.c_int32), ("reserved", ctypes.c_int32),
    ]

    def as_dict(self):
        d = {name: getattr(self, name) for name, _ in self._fields_}
        d["phase_cycles"] = list(d["phase_cycles"])
        return d


_SIGS = {
    "bang_last_error": (ctypes.c_char_p, []),
    "bang_version": (ctypes.c_char_p, []),
    "bang_device_count": (_I32, []),
    "bang_index_create": (_I32, [_I32, _P, _I64, _I32, _P, _P, _I32, _P, _P, _I32, _I32, _P,
                                 _I32, _I32, ctypes.POINTER(_P)]),
    "bang_index_destroy": (None, [_P]),
    "bang_read_graph_header": (_I32, [ctypes.c_char_p, _P, _P, _P]),
    "bang_read_graph": (_I32, [ctypes.c_char_p, _P, _P, _I64, _I32, _I32]),
    "bang_index_info": (_I32, [_P, _P, _P, _P, _P, _P]),
    "bang_index_device_ptrs": (_I32, [_P, _P, _P, _P, _P, _P]),
    "bang_index_code_stride": (_I32, [_P]),
    "bang_index_prepare": (_I32, [_P, _I64]),
    "bang_options_default": (None, [ctypes.POINTER(Options)]),
    "bang_index_set_options": (_I32, [_P, ctypes.POINTER(Options)]),
    "bang_index_get_options": (_I32, [_P, ctypes.POINTER(Options)]),
    "bang_pq_table": (_I32, [_P, _P, _I64, _P]),
    "bang_search": (_I32, [_P, _P, _I64, _I32, _I32, _I64, _I32, _P, _P, _P, _P, _P, _P, _P,
                           _P, _I64]),
    "bang_last_visit_logs": (_I32, [_P, _P, _I64]),
    "bang_last_search_stats": (_I32, [_P, ctypes.POINTER(SearchStats)]),
    "bang_index_set_log_capacity": (_I32, [_P, _I64]),
    "bang_search_device": (_I32, [_P, _P, _I64, _I32, _I32, _I64, _I32, _P, _P, _P, _P, _P]),
    "bang_sync_status": (_I32, [_P]),
    "bang_pq_table_device": (_I32, [_P, _P, _I32, _I32, _P, _I64, _P, _P]),
    "bang_bloom_filter_device": (_I32, [_P, _I64, _I64, _P, _P, _P, _P]),
    "bang_adc_device": (_I32, [_P, _I32, _P, _P, _P, _I64, _P, _P, _P]),
    "bang_adc_pairs_device": (_I32, [_P, _P, _I64, _P, _P, _P, _P]),
    "bang_sort_rows_device": (_I32, [_P, _I64, _I32, _P]),
    "bang_merge_rows_device": (_I32, [_P, _P, _I64, _I32, _P, _I32, _P, _P, _P]),
    "bang_worklist_update_device": (_I32, [_P, _P, _I64, _I32, _P, _I32, _P, _P, _P]),
    "bang_rerank_device": (_I32, [_P, _I32, _I32, _P, _I64, _P, _P, _I32, _P, _P, _P, _P]),
    "bang_exact_sq_dists_device": (_I32, [_P, _I32, _I32, _P, _I64, _P, _P]),
    "bang_host_read_bandwidth": (_I32, [_I32, _I64, _I32, _I32, ctypes.POINTER(ctypes.c_double)]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """Load libbang.so once; raise BangError if it is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise BangError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                            "(there is no CPU fallback for the search path)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().bang_last_error().decode("utf-8", "replace")


def check(status: int, what: str = "") -> None:
    """Map a bang_status onto the reference's exception classes."""
    if status == BANG_OK:
        return
    msg = last_error() or what
    if status == BANG_E_PARAM:
        raise ParameterError(msg)
    if status == BANG_E_FORMAT:
        raise FileFormatError(msg)
    if status == BANG_E_TRUNCATED:
        raise TruncatedFileError(msg)
    raise BangError(f"{what}: {msg} (status {status})" if what else msg)


def device_count() -> int:
    return int(lib().bang_device_count())


def ptr(a):
    """Raw address of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return ctypes.c_void_p(a.data_ptr())
    return a.ctypes.data_as(ctypes.c_void_p)


def stream_ptr(stream):
    if stream is None:
        return None
    return ctypes.c_void_p(int(getattr(stream, "cuda_stream", stream)))
