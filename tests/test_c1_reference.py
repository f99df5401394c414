"""BASELINE config C1 pinned against the reference itself.

tests/golden/c1_reference.npz holds the reference's own artifacts and
outputs for configs[0] (make_c1.py: datasets.gaussian_mixture, VamanaBuilder
R=32 L=64, ProductQuantizer m=32, GraphSearcher.search at t=48 and t=152).
The base vectors are regenerated from the seed and checked by SHA-256.
CPU tests: the generator and the oracle reproduce the reference; GPU tests:
libbang.so reproduces it bit for bit (visit logs, iterations, ids, dists).
"""

import hashlib

import numpy as np
import pytest

import golden_util as gu
from oracle import oracle as O

_C1 = {}


def c1():
    if not _C1:
        from paper_2401_11324_b200.tools.datasets import gaussian_mixture
        g = gu.load("c1_reference.npz")
        base, q = gaussian_mixture(int(g["n"]), g["queries"].shape[0], int(g["dim"]), clusters=int(g["clusters"]),
                                   seed=int(g["seed"]))
        g["base"] = base
        g["regen_queries"] = q
        _C1.update(g)
    return _C1


def _refs(g, t):
    return (g[f"t{t}_ids"], g[f"t{t}_dists"], g[f"t{t}_iterations"],
            gu.logs(g[f"t{t}_log_offsets"], g[f"t{t}_log_ids"]), g[f"t{t}_short"])


def test_c1_generator_reproduces_reference_data():
    g = c1()
    assert hashlib.sha256(np.ascontiguousarray(g["base"]).tobytes()).hexdigest() == str(g["base_sha256"])
    assert np.array_equal(g["regen_queries"], g["queries"])
    assert hashlib.sha256(g["queries"].tobytes()).hexdigest() == str(g["queries_sha256"])


@pytest.mark.parametrize("t", [48, 152])
def test_c1_oracle_matches_reference(t):
    g = c1()
    cents = gu.split_centroids(g["centroids"], g["sub_sizes"])
    want_ids, want_d, want_it, want_logs, want_short = _refs(g, t)
    got = O.search(g["queries"], centroids=cents, sub_sizes=g["sub_sizes"], codes=g["codes"],
                   adjacency=g["adjacency"], degrees=g["degrees"], medoid=int(g["medoid"]), vectors=g["base"],
                   k=int(g["k"]), t=t, bloom_entries=int(g["bloom_entries"]), threads=8)
    assert np.array_equal(got["iterations"], want_it)
    for a, b in zip(got["visit_logs"], want_logs):
        assert np.array_equal(a, b)
    assert np.array_equal(got["ids"], want_ids)
    assert np.array_equal(got["dists"], want_d)
    assert np.array_equal(got["short"], want_short)


@pytest.mark.gpu
@pytest.mark.parametrize("t", [48, 152])
@pytest.mark.parametrize("kernel,variant", [("auto", "auto"), ("cta", "auto"), ("warp", "smem-table"),
                                            ("warp", "codebook")])
def test_c1_gpu_matches_reference(t, kernel, variant):
    B = pytest.importorskip("paper_2401_11324_b200")
    g = c1()
    cents = gu.split_centroids(g["centroids"], g["sub_sizes"])
    cb = B.PQCodebook(dim=int(g["dim"]), subspace_sizes=[int(s) for s in g["sub_sizes"]], centroids=cents)
    graph = B.GraphIndex(g["adjacency"], g["degrees"], int(g["medoid"]), int(g["degree_bound"]))
    s = B.GraphSearcher(k=int(g["k"]), t=t, mode="in_memory", bloom_entries=int(g["bloom_entries"]),
                        debug_checks=True)
    s.fit(g["base"], graph=graph, codebook=cb, codes=B.CompressedVectors(g["codes"]))
    res = s.set_kernel(kernel).set_adc_variant(variant).search(g["queries"])
    want_ids, want_d, want_it, want_logs, want_short = _refs(g, t)
    assert np.array_equal(res.iterations, want_it)
    for a, b in zip(res.visit_logs, want_logs):
        assert np.array_equal(a, b)
    assert np.array_equal(res.ids, want_ids)
    assert np.array_equal(res.dists, want_d)
    assert np.array_equal(res.short, want_short)
    if kernel == "auto":
        assert s.last_stats()["kernel"] == 8  # HBM graph, m = 32: search_split_kernel
