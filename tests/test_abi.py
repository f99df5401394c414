"""The C-ABI library loads and exports every entry point include/bang.h
declares; with no GPU visible it fails loudly instead of falling back."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2401_11324_b200 import _lib
from paper_2401_11324_b200.errors import BangError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "bang.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bang_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_expected_surface():
    names = _declared()
    for n in ("bang_index_create", "bang_search", "bang_pq_table_device", "bang_bloom_filter_device",
              "bang_adc_device", "bang_worklist_update_device", "bang_rerank_device"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_declared()) == set(_lib.EXPORTED)


def test_version_and_error_strings():
    assert _lib.lib().bang_version().startswith(b"bang-b200")
    assert isinstance(_lib.last_error(), str)


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    assert _lib.device_count() == 0
    h = ctypes.c_void_p()
    adj = np.zeros((2, 1), np.int32)
    adj[0, 0], adj[1, 0] = 1, 0
    deg = np.ones(2, np.int32)
    vec = np.zeros((2, 2), np.float32)
    st = _lib.lib().bang_index_create(0, None, 2, 0, None, None, 2, _lib.ptr(adj), _lib.ptr(deg), 1, 0,
                                      _lib.ptr(vec), 0, 0, ctypes.byref(h))
    assert st != 0 and not h.value
    with pytest.raises(BangError):
        _lib.check(st, "bang_index_create")


def test_parameter_errors_map_to_parameter_error():
    from paper_2401_11324_b200.errors import ParameterError
    st = _lib.lib().bang_index_create(0, None, 0, 0, None, None, 2, None, None, 1, 0, None, 0, 0,
                                      ctypes.byref(ctypes.c_void_p()))
    assert st == _lib.BANG_E_PARAM
    with pytest.raises(ParameterError):
        _lib.check(st)
