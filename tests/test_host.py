"""Host-side logic of the drop-in API (no GPU): validation, parameter
checks, key packing, Bloom slot hashing, index-load readers/writers."""

import numpy as np
import pytest

import golden_util as gu
import paper_2401_11324_b200 as B
from paper_2401_11324_b200.engine import GraphSearcher


def _toy_graph():
    g = gu.load("search_toy_k2.npz")
    return g, B.GraphIndex(g["adjacency"], g["degrees"], int(g["medoid"]), int(g["degree_bound"]))


def test_constructor_params_mirror_reference():
    s = GraphSearcher()
    p = s.get_params()
    assert p == dict(k=10, t=152, mode="pipelined", bloom_entries=399_887, batch_size=10_000, rerank=True,
                     degree_bound=64, build_worklist=200, sigma=1.2, m=74, pq_iters=25, seed=0,
                     threads=None, debug_checks=False)
    from sklearn.base import clone
    assert clone(GraphSearcher(k=3, t=9)).get_params()["t"] == 9


@pytest.mark.parametrize("kw", [dict(k=10, t=5), dict(mode="warp"), dict(bloom_entries=0),
                                dict(batch_size=0), dict(k=0)])
def test_invalid_params_rejected_before_any_device_work(kw):
    g, graph = _toy_graph()
    with pytest.raises(B.ParameterError):
        GraphSearcher(**kw).fit(g["base"], graph=graph)


def test_search_before_fit_raises():
    with pytest.raises(B.ParameterError):
        GraphSearcher().search(np.zeros((1, 2), np.float32))


def test_check_matrix_rejects_nan():
    from paper_2401_11324_b200.validation import check_matrix
    with pytest.raises(B.ParameterError):
        check_matrix(np.array([[np.nan, 1.0]]))
    with pytest.raises(B.ParameterError):
        check_matrix(np.zeros((2, 2, 2)))


def test_pack_unpack_and_order():
    rng = np.random.default_rng(1)
    d = np.repeat(rng.random(200).astype(np.float32), 2)
    ids = rng.permutation(400)
    keys = B.pack_keys(d, ids)
    assert np.array_equal(np.argsort(keys), np.lexsort((ids, d)))
    dd, ii = B.unpack_keys(keys)
    assert np.array_equal(dd, d) and np.array_equal(ii, ids)
    assert int(B.pack_keys(np.float32([73.0]), [10])[0]) == 0x429200000000000A


def test_bloom_slots_match_reference_golden():
    g = gu.load("bloom.npz")
    p1, p2 = B.bit_positions(g["pin_ids"], 399_887)
    assert np.array_equal(p1, g["pin_p1"]) and np.array_equal(p2, g["pin_p2"])


def test_subspace_split():
    assert B.subspace_split(128, 74) == [2] * 54 + [1] * 20
    assert B.subspace_split(7, 3) == [3, 2, 2]
    with pytest.raises(B.ParameterError):
        B.subspace_split(4, 5)


def test_graph_validation():
    with pytest.raises(B.ParameterError):
        B.GraphIndex.from_lists([[0]], medoid=0, degree_bound=1)  # self loop
    with pytest.raises(B.ParameterError):
        B.GraphIndex.from_lists([[1, 1], [0]], medoid=0, degree_bound=2)  # duplicate
    with pytest.raises(B.ParameterError):
        B.GraphIndex.from_lists([[1], [0]], medoid=5, degree_bound=1)


def test_graph_codebook_codes_roundtrip(tmp_path):
    g = gu.load("search_random_r64.npz")
    graph = B.GraphIndex(g["adjacency"], g["degrees"], int(g["medoid"]), int(g["degree_bound"]))
    B.write_graph(graph, str(tmp_path / "g.pgix"))
    back = B.read_graph(str(tmp_path / "g.pgix"))
    assert back == graph
    cb = B.PQCodebook(dim=g["base"].shape[1], subspace_sizes=[int(s) for s in g["sub_sizes"]],
                      centroids=gu.split_centroids(g["centroids"], g["sub_sizes"]))
    B.write_codebook(cb, str(tmp_path / "c.pqcb"))
    assert B.read_codebook(str(tmp_path / "c.pqcb")) == cb
    codes = B.CompressedVectors(g["codes"])
    B.write_codes(codes, str(tmp_path / "c.pqcv"))
    assert np.array_equal(B.read_codes(str(tmp_path / "c.pqcv")).codes, codes.codes)
    for fmt, arr in (("fvecs", g["base"]), ("raw_bin", g["base"]),
                     ("bvecs", (np.abs(g["base"]) * 10).astype(np.uint8))):
        B.write_vectors(B.VectorStore(arr), str(tmp_path / f"v.{fmt}"), fmt)
        assert np.array_equal(B.read_vectors(str(tmp_path / f"v.{fmt}"), fmt).data, arr)


def test_graph_reader_rejects_corruption(tmp_path):
    g, graph = _toy_graph()
    p = tmp_path / "g.pgix"
    B.write_graph(graph, str(p))
    raw = p.read_bytes()
    (tmp_path / "t.pgix").write_bytes(raw[:-2])
    with pytest.raises((B.TruncatedFileError, B.FileFormatError)):
        B.read_graph(str(tmp_path / "t.pgix"))
    (tmp_path / "x.pgix").write_bytes(raw + b"\0\0\0\0")
    with pytest.raises((B.FileFormatError, B.TruncatedFileError)):
        B.read_graph(str(tmp_path / "x.pgix"))
    (tmp_path / "m.pgix").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(B.FileFormatError):
        B.read_graph(str(tmp_path / "m.pgix"))


def test_reference_graph_file_is_read_identically(tmp_path):
    """A file written in the reference's PGIX layout (io.py:242-251)."""
    import struct
    lists = [[1, 2], [], [0]]
    blob = b"PGIX" + struct.pack("<4I", 1, 3, 2, 0)
    for ids in lists:
        blob += struct.pack("<I", len(ids)) + struct.pack(f"<{len(ids)}I", *ids)
    (tmp_path / "r.pgix").write_bytes(blob)
    graph = B.read_graph(str(tmp_path / "r.pgix"))
    assert graph.degrees.tolist() == [2, 0, 1]
    assert graph.adjacency.tolist() == [[1, 2], [-1, -1], [0, -1]]


def test_dataset_generator_matches_reference_stream():
    from paper_2401_11324_b200.tools.datasets import gaussian_mixture
    g = gu.load("search_vamana_f32.npz")
    base, q = gaussian_mixture(3000, 48, 16, clusters=24, seed=101)
    assert np.array_equal(base, g["base"]) and np.array_equal(q, g["queries"])


def test_native_graph_reader_matches_reference_cases(tmp_path):
    """bang_read_graph (native, mmap) against the reference reader's outcome
    on valid and corrupted PGIX files (tests/golden/make_io_golden.py): the
    same arrays, or the same exception class and message."""
    g = gu.load("io_graph_cases.npz")
    for name in [str(v) for v in g["names"]]:
        path = tmp_path / f"{name}.pgix"
        path.write_bytes(g[f"{name}__bytes"].tobytes())
        if f"{name}__error" in g:
            cls = getattr(B, str(g[f"{name}__error"]))
            with pytest.raises(cls) as ei:
                B.read_graph(str(path))
            assert type(ei.value).__name__ == str(g[f"{name}__error"]), name
            assert str(ei.value) == str(g[f"{name}__message"]).replace("{path}", str(path)), name
        else:
            got = B.read_graph(str(path))
            assert np.array_equal(got.adjacency, g[f"{name}__adjacency"]), name
            assert np.array_equal(got.degrees, g[f"{name}__degrees"]), name
            assert got.medoid == int(g[f"{name}__medoid"]), name


def test_native_graph_reader_threads_agree(tmp_path):
    """Thread count never changes the result (the copy pass is partitioned by node)."""
    rng = np.random.default_rng(3)
    n, R = 20_000, 24
    deg = rng.integers(0, R + 1, size=n).astype(np.int32)
    adj = np.full((n, R), -1, np.int32)
    for i in range(n):
        ids = rng.choice(n - 1, size=int(deg[i]), replace=False)
        adj[i, :deg[i]] = ids + (ids >= i)
    graph = B.GraphIndex(adj, deg, 7, R)
    B.write_graph(graph, str(tmp_path / "g.pgix"))
    for threads in (1, 3, 0):
        assert B.read_graph(str(tmp_path / "g.pgix"), threads=threads) == graph
