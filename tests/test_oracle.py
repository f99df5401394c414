"""Pin the CPU oracle (oracle/bang_oracle.c) to the reference's own outputs.

The golden fixtures were produced by the reference itself
(tests/golden/make_golden.py).  If these pass, the oracle restates the
reference bit-for-bit on every case, and the GPU parity tests may use the
oracle as their checker at sizes the fixtures do not cover.
"""

import numpy as np
import pytest

import golden_util as gu
from oracle import oracle as O


def test_pq_table_matches_reference_exactly():
    g = gu.load("pq_table.npz")
    for tag in "abcd":
        cents = gu.split_centroids(g[f"{tag}_centroids"], g[f"{tag}_sizes"])
        got = O.pq_table(g[f"{tag}_q"], cents, g[f"{tag}_sizes"])
        assert np.array_equal(got, g[f"{tag}_table"]), tag


def test_adc_matches_reference_exactly():
    g = gu.load("adc.npz")
    got = O.adc(g["table"], g["codes"], g["qrows"], g["ids"])
    assert np.array_equal(got, g["dists"])
    assert np.array_equal(O.pack_keys(got, g["ids"]), g["keys"])


def test_bloom_pinned_slots():
    g = gu.load("bloom.npz")
    p1, p2 = O.bit_positions(g["pin_ids"], 399_887)
    assert np.array_equal(p1, g["pin_p1"]) and np.array_equal(p2, g["pin_p2"])
    # SURVEY.md 8(c) computed from bloom.py: id 0 -> (42984, 386527)
    assert (int(p1[0]), int(p2[0])) == (42984, 386527)
    assert O.lib().bo_fnv1a(0, 0) == 0x4D25767F9DCE13F5
    assert O.lib().bo_fnv1a(0, 1) == 0x5A382CC93317501D


@pytest.mark.parametrize("case", range(5))
def test_bloom_bank_sequences_match_reference(case):
    g = gu.load("bloom.npz")
    count, entries = int(g[f"c{case}_count"]), int(g[f"c{case}_entries"])
    bits = np.zeros((count, (entries + 63) // 64), np.uint64)
    sp = g[f"c{case}_splits"]
    for a, b in zip(sp[:-1], sp[1:]):
        fr = O.bloom_filter_and_set(bits, entries, g[f"c{case}_rows"][a:b], g[f"c{case}_ids"][a:b])
        assert np.array_equal(fr, g[f"c{case}_fresh"][a:b])
    assert np.array_equal(bits, g[f"c{case}_bits"])


def test_sort_and_merge_rows_match_reference():
    g = gu.load("kernels.npz")
    assert np.array_equal(O.sort_rows(g["keys"]), g["sorted"])
    mk, mp = O.merge_rows(g["a"], g["b"], a_payload=g["a_payload"])
    assert np.array_equal(mk, g["merged"]) and np.array_equal(mp, g["merged_payload"])


def test_exact_distances_and_rerank_match_reference():
    g = gu.load("exact.npz")
    assert np.array_equal(O.exact_sq_dists(g["x"], g["q"]), g["ex"])
    assert np.array_equal(O.exact_sq_dists(g["xu"], g["qu"]), g["exu"])


@pytest.mark.parametrize("name", gu.search_cases())
def test_search_matches_reference(name):
    g = gu.load(name)
    res = O.search(g["queries"], centroids=gu.split_centroids(g["centroids"], g["sub_sizes"]),
                   sub_sizes=g["sub_sizes"], codes=g["codes"], adjacency=g["adjacency"],
                   degrees=g["degrees"], medoid=int(g["medoid"]), vectors=g["base"],
                   k=int(g["k"]), t=int(g["t"]), bloom_entries=int(g["bloom_entries"]),
                   rerank=bool(g["rerank"]), threads=4)
    assert np.array_equal(res["iterations"], g["iterations"])
    for got, want in zip(res["visit_logs"], gu.logs(g["log_offsets"], g["log_ids"])):
        assert np.array_equal(got, want)
    assert np.array_equal(res["ids"], g["ids"])
    assert np.array_equal(res["dists"], g["dists"])
    assert np.array_equal(res["short"], g["short"])
    assert np.array_equal(res["converged"], g["converged"])
    if "ex_ids" in g:  # exact_distance mode (engine.py:120-124, 188-193)
        ex = O.search(g["queries"], centroids=None, sub_sizes=None, codes=None,
                      adjacency=g["adjacency"], degrees=g["degrees"], medoid=int(g["medoid"]),
                      vectors=g["base"], k=int(g["k"]), t=int(g["t"]),
                      bloom_entries=int(g["bloom_entries"]), mode="exact")
        assert np.array_equal(ex["ids"], g["ex_ids"])
        assert np.array_equal(ex["dists"], g["ex_dists"])
        assert np.array_equal(ex["iterations"], g["ex_iterations"])
        for got, want in zip(ex["visit_logs"], gu.logs(g["ex_log_offsets"], g["ex_log_ids"])):
            assert np.array_equal(got, want)


def test_toy_trace_constants():
    # conftest.py:53-54 of the reference: the paper's Fig. 2 worked example
    g = gu.load("search_toy_k2.npz")
    assert g["log_ids"].tolist() == [6, 8, 7, 2, 5, 9, 11, 10]
    assert set(g["ids"][0].tolist()) == {10, 8}
    g8 = gu.load("search_toy_k8.npz")
    assert g8["ids"][0].tolist() == [10, 8, 11, 9, 6, 7, 5, 2]
