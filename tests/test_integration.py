"""The reference-side binding (integration/bang_gpu.py, the bang/_gpu.py of
INTEGRATION.md) executed for real.

The module uses only names the reference package defines; it is loaded here
as a submodule of paper_2401_11324_b200 (whose errors/graph/pq classes carry
the same names), so its relative import resolves without touching the
read-only reference.  GPU tests compare its search and table outputs with
fixtures the reference itself produced; the CPU tests run the native loader
through it and, where the reference is present, check that the seam it
replaces still has the cited shape.
"""

import importlib.util
import inspect
import os
import sys

import numpy as np
import pytest

import golden_util as gu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BINDING = os.path.join(ROOT, "integration", "bang_gpu.py")
REF_SRC = "/root/reference/pkg/src"


def _binding():
    import paper_2401_11324_b200 as B
    from paper_2401_11324_b200 import _lib
    os.environ.setdefault("BANG_LIBBANG", _lib.LIB_PATH)
    name = "paper_2401_11324_b200._ref_gpu_binding"
    if name in sys.modules:
        return B, sys.modules[name]
    spec = importlib.util.spec_from_file_location(name, BINDING)
    mod = importlib.util.module_from_spec(spec)
    mod.__package__ = "paper_2401_11324_b200"
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return B, mod


def test_binding_reads_graphs_like_the_reference(tmp_path):
    B, G = _binding()
    g = gu.load("io_graph_cases.npz")
    for name in [str(v) for v in g["names"]]:
        p = tmp_path / f"{name}.pgix"
        p.write_bytes(g[f"{name}__bytes"].tobytes())
        if f"{name}__error" in g and str(g[f"{name}__error"]) in ("FileFormatError", "TruncatedFileError"):
            with pytest.raises(getattr(B, str(g[f"{name}__error"]))) as ei:
                G.read_graph_arrays(str(p))
            assert str(ei.value) == str(g[f"{name}__message"]).replace("{path}", str(p))
        elif f"{name}__adjacency" in g:
            adj, deg, med, R = G.read_graph_arrays(str(p))
            assert np.array_equal(adj, g[f"{name}__adjacency"]) and np.array_equal(deg, g[f"{name}__degrees"])
            assert med == int(g[f"{name}__medoid"])


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference sources not present (GPU box)")
def test_reference_seam_has_the_hooked_shape():
    """The two hook points INTEGRATION.md names exist with the signatures the
    binding reproduces (engine.py:108-112 _search_batch, engine.py:377-452)."""
    import subprocess
    code = (
        "import inspect, sys; sys.dont_write_bytecode = True; sys.path.insert(0, %r)\n"
        "from bang import engine\n"
        "sig = inspect.signature(engine._search_batch)\n"
        "print(','.join(sig.parameters))\n"
        "print(','.join(inspect.signature(engine.GraphSearcher.fit).parameters))\n"
    ) % REF_SRC
    env = dict(os.environ, NUMBA_CACHE_DIR="/tmp/numba_cache", PYTHONDONTWRITEBYTECODE="1")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, check=True)
    params, fit = out.stdout.strip().splitlines()
    assert params.split(",")[:2] == ["host", "queries"]
    for kw in ("k", "t", "mode", "bloom_entries", "table", "debug_checks"):
        assert kw in params.split(",")
    assert fit.split(",")[:3] == ["self", "X", "y"] and {"graph", "codebook", "codes"} <= set(fit.split(","))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["search_vamana_f32.npz", "search_vamana_u8.npz", "search_random_r64.npz",
                                  "search_vamana_norerank.npz"])
def test_binding_search_matches_reference_fixture(name):
    B, G = _binding()
    g = gu.load(name)
    cb = B.PQCodebook(dim=g["base"].shape[1], subspace_sizes=[int(s) for s in g["sub_sizes"]],
                      centroids=gu.split_centroids(g["centroids"], g["sub_sizes"]))
    graph = B.GraphIndex(g["adjacency"], g["degrees"], int(g["medoid"]), int(g["degree_bound"]))
    idx = G.GpuIndex(graph, g["base"], cb, B.CompressedVectors(g["codes"]))
    ids, dists, it, conv, wall, short, logs = idx.search_batch(g["queries"], int(g["k"]), int(g["t"]),
                                                               int(g["bloom_entries"]), bool(g["rerank"]), True)
    assert np.array_equal(ids, g["ids"]) and np.array_equal(dists, g["dists"])
    assert np.array_equal(it, g["iterations"]) and conv.all()
    offs = g["log_offsets"]
    for i, lg in enumerate(logs):
        assert np.array_equal(lg, g["log_ids"][offs[i]:offs[i + 1]])
    idx.close()


@pytest.mark.gpu
def test_binding_pq_table_and_errors():
    B, G = _binding()
    g = gu.load("pq_table.npz")
    cents = gu.split_centroids(g["b_centroids"], g["b_sizes"])
    cb = B.PQCodebook(dim=g["b_q"].shape[1], subspace_sizes=[int(s) for s in g["b_sizes"]], centroids=cents)
    n = 16
    rng = np.random.default_rng(0)
    graph = B.GraphIndex.from_lists([[(i + 1) % n] for i in range(n)], medoid=0, degree_bound=1)
    base = rng.normal(size=(n, cb.dim)).astype(np.float32)
    codes = B.CompressedVectors(rng.integers(0, 256, size=(n, cb.m), dtype=np.uint8))
    idx = G.GpuIndex(graph, base, cb, codes)
    assert np.array_equal(idx.pq_table(g["b_q"]), g["b_table"])
    with pytest.raises(B.ParameterError):
        idx.search_batch(base[:2], 5, 4, 399_887)  # k > t
    idx.close()
