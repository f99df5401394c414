"""Offline tooling on the CPU (torch CPU tensors): the partitioned k-NN and
search-based Vamana pass used for the 10M-point benchmark graph, the chunked
data generator, the artifact cache, and the CSR visit-log view.  None of this
is the search path; it builds the benchmark's inputs."""

import os

import numpy as np
import pytest

from paper_2401_11324_b200.engine import VisitLogs
from paper_2401_11324_b200.tools import graph_build as gb
from paper_2401_11324_b200.tools.datasets import gaussian_mixture


def _exact_knn(x, K):
    d = ((x[:, None, :].astype(np.float64) - x[None, :, :]) ** 2).sum(-1)
    np.fill_diagonal(d, np.inf)
    return np.argsort(d, 1, kind="stable")[:, :K]


def test_knn_ivf_finds_most_true_neighbours():
    import torch
    b, _ = gaussian_mixture(3000, 0, 16, clusters=30, seed=1)
    ids, d = gb.knn_ivf(torch.from_numpy(b), 20, nlist=12, nprobe=6, seed=0)
    ids = ids.numpy()
    assert ids.shape == (3000, 20)
    assert (ids != np.arange(3000)[:, None]).all()          # self excluded
    assert np.isfinite(d.numpy()[ids >= 0]).all()
    want = _exact_knn(b, 20)
    rec = np.mean([len(set(a) & set(w)) / 20 for a, w in zip(ids, want)])
    assert rec > 0.8


def test_robust_prune_keeps_nearest_and_respects_degree():
    import torch
    b, _ = gaussian_mixture(800, 0, 8, clusters=8, seed=2)
    x = torch.from_numpy(b)
    ids, d = gb.knn(x, 32)
    ids, d = gb._sort_rows_by_dist(ids, d)
    adj, deg = gb.robust_prune(x, ids, d, 12, 1.2)
    adj, deg = adj.numpy(), deg.numpy()
    assert (deg >= 1).all() and (deg <= 12).all()
    assert (adj[:, 0] == ids.numpy()[:, 0]).all()             # the nearest is always kept
    for i in range(0, 800, 37):
        row = adj[i, :deg[i]]
        assert (row >= 0).all() and len(set(row.tolist())) == deg[i] and i not in row
        assert (adj[i, deg[i]:] == -1).all()


def test_refine_pass_with_oracle_search_builds_a_valid_graph():
    """One batch-synchronous Vamana pass driven by the oracle's visit logs."""
    import torch
    from oracle import oracle as O
    from paper_2401_11324_b200.tools.pq_train import encode, train_codebook
    b, q = gaussian_mixture(2000, 100, 16, clusters=20, seed=3)
    x = torch.from_numpy(b)
    g0 = gb.build_graph(b, 16, device="cpu", exact_limit=100)   # IVF path
    cb = train_codebook(b, m=4, iters=4, seed=0, device="cpu")
    codes = encode(b, cb, device="cpu").codes
    A, D = g0.adjacency, g0.degrees

    def visit_fn(lo, hi):
        r = O.search(b[lo:hi], centroids=cb.centroids, sub_sizes=cb.subspace_sizes, codes=codes,
                     adjacency=A, degrees=D, medoid=g0.medoid, vectors=b, k=5, t=24,
                     bloom_entries=399_887, threads=4)
        logs = r["visit_logs"]
        offs = np.concatenate([[0], np.cumsum([len(l) for l in logs])])
        return offs, np.concatenate(logs)

    adj, deg = gb.refine_graph(x, torch.from_numpy(A).long(), torch.from_numpy(D).long(), visit_fn, 16,
                               chunk=700)
    adj, deg = adj.numpy(), deg.numpy()
    assert (deg >= 1).all() and (deg <= 16).all()
    assert all(i not in adj[i, :deg[i]] for i in range(2000))
    assert (adj[np.arange(16)[None, :] >= deg[:, None]] == -1).all()


def test_chunked_generator_equals_one_shot_stream():
    a, qa = gaussian_mixture(3000, 50, 12, clusters=7, seed=9)
    rng = np.random.default_rng(9)
    axis = (np.arange(12) + 1.0) ** -0.5
    centers = rng.normal(0.0, 1.0, size=(7, 12)) * axis
    which = rng.integers(0, 7, size=3000)
    want = (centers[which] + rng.normal(0.0, 1.0, size=(3000, 12)) * axis).astype(np.float32)
    assert np.array_equal(a, want)


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src/bang"), reason="reference not mounted")
def test_generator_matches_reference_datasets_module():
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        from bang.datasets import gaussian_mixture as ref
    except Exception as e:  # pragma: no cover
        pytest.skip(f"reference import failed: {e}")
    rb, rq = ref(2500, 40, 24, clusters=11, seed=4)
    b, q = gaussian_mixture(2500, 40, 24, clusters=11, seed=4)
    assert np.array_equal(np.asarray(rb.data), b) and np.array_equal(np.asarray(rq.data), q)


def test_visit_logs_csr_roundtrip():
    parts = [(np.array([0, 2, 2, 5]), np.array([4, 1, 7, 8, 9])), (np.array([0, 1]), np.array([3]))]
    v = VisitLogs(parts)
    offs, flat = v.csr()
    assert offs.tolist() == [0, 2, 2, 5, 6] and flat.tolist() == [4, 1, 7, 8, 9, 3]
    assert [x.tolist() for x in v] == [[4, 1], [], [7, 8, 9], [3]]


def test_artifact_cache_roundtrip(tmp_path):
    from paper_2401_11324_b200.graph import GraphIndex
    from paper_2401_11324_b200.pq import CompressedVectors, PQCodebook
    from paper_2401_11324_b200.tools import bench_data as bd
    rng = np.random.default_rng(0)
    arrays = dict(base=rng.random((10, 4), dtype=np.float32), queries=rng.random((3, 4), dtype=np.float32),
                  adjacency=np.full((10, 2), -1, np.int32), degrees=np.zeros(10, np.int32), medoid=np.int64(3),
                  sub_sizes=np.array([2, 2], np.int32), centroids=rng.random(1024, dtype=np.float32),
                  codes=rng.integers(0, 256, (10, 2), dtype=np.uint8), gt_ids=np.zeros((3, 10), np.int32),
                  gt_dists=np.zeros((3, 10), np.float32))
    path = str(tmp_path / "c")
    bd._save_cached(path, arrays, log=lambda *a: None)
    meta = dict(desc="t", n=10, dim=4, dtype="f32", R=2, m=2, clusters=1)
    art = bd._load_cached(path, "T", meta, log=lambda *a: None)
    assert np.array_equal(np.asarray(art["base"]), arrays["base"])
    assert isinstance(art["graph"], GraphIndex) and art["graph"].medoid == 3
    assert isinstance(art["codebook"], PQCodebook) and art["codebook"].centroids[1].shape == (256, 2)
    assert isinstance(art["codes"], CompressedVectors)


def test_locality_order_relabel_is_an_isomorphism():
    """graph_build.locality_order + relabel_index rename nodes only: every
    edge, degree, vector and the medoid survive under the permutation, and
    nodes of one k-means cell end up contiguous."""
    import torch
    base, _ = gaussian_mixture(3_000, 0, 16, clusters=30, seed=4)
    g = gb.build_graph(base, degree_bound=12, seed=4, device=torch.device("cpu"))
    perm = gb.locality_order(base, nlist=8, seed=4, device=torch.device("cpu"))
    assert np.array_equal(np.sort(perm), np.arange(base.shape[0]))
    b2, adj2, deg2, med2 = gb.relabel_index(perm, base, g.adjacency, g.degrees, g.medoid,
                                            device=torch.device("cpu"))
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    assert np.array_equal(b2, base[perm]) and np.array_equal(deg2, g.degrees[perm])
    assert med2 == inv[g.medoid]
    for new in range(0, perm.size, 97):
        old = perm[new]
        d = g.degrees[old]
        assert np.array_equal(adj2[new, :d], inv[g.adjacency[old, :d]])
        assert np.all(adj2[new, d:] == -1)


def test_partitioned_build_is_valid_and_as_good_as_monolithic():
    """build_graph_partitioned (the C4 builder): a valid GraphIndex (no self
    loops or duplicates, -1 padding past the degree) whose exact-distance
    greedy search recall matches the one-shot build on the same data."""
    from oracle import oracle as O
    b, q = gaussian_mixture(12_000, 100, 16, clusters=120, seed=4, out_dtype=np.uint8)
    qf = q.astype(np.float32)
    gp = gb.build_graph_partitioned(b, degree_bound=16, parts=4, overlap=2, device="cpu", merge_chunk=3000)
    gp.validate()
    assert gp.degrees.min() >= 1
    gm = gb.build_graph(b, degree_bound=16, device="cpu")
    d = ((qf[:, None, :].astype(np.float64) - b[None, :, :].astype(np.float64)) ** 2).sum(-1)
    gt = np.argsort(d, 1, kind="stable")[:, :10]

    def rec(g):
        r = O.search(qf, centroids=None, sub_sizes=None, codes=None, adjacency=g.adjacency, degrees=g.degrees,
                     medoid=g.medoid, vectors=b, k=10, t=32, bloom_entries=399_887, mode="exact", threads=4)
        return np.mean([len(set(a) & set(c)) / 10 for a, c in zip(r["ids"], gt)])

    assert rec(gp) >= rec(gm) - 0.03


def test_partitioned_build_resumes_from_checkpoint(tmp_path):
    """The C4 builder checkpoints the assignment, the candidate table and each
    finished partition: a run stopped after some partitions resumes and gives
    the graph of an uninterrupted run (one device, deterministic CPU ops)."""
    b, _ = gaussian_mixture(6_000, 0, 16, clusters=60, seed=5, out_dtype=np.uint8)
    full = gb.build_graph_partitioned(b, degree_bound=12, parts=3, overlap=2, device="cpu", merge_chunk=2000,
                                      ckpt_dir=str(tmp_path / "a"))
    ck = tmp_path / "b"
    ck.mkdir()
    calls = []

    def stop_after_two(members, g, t):
        calls.append(t)
        if len(calls) == 3:
            raise KeyboardInterrupt  # the session ends during partition 3
        return g
    with pytest.raises(KeyboardInterrupt):
        gb.build_graph_partitioned(b, degree_bound=12, parts=3, overlap=2, device="cpu", merge_chunk=2000,
                                   refine_fn=stop_after_two, refine=(1,), ckpt_dir=str(ck))
    assert open(ck / "done.txt").read().split() == ["0", "1"]
    redo = []
    resumed = gb.build_graph_partitioned(b, degree_bound=12, parts=3, overlap=2, device="cpu", merge_chunk=2000,
                                         refine_fn=lambda m, g, t: redo.append(t) or g, refine=(1,),
                                         ckpt_dir=str(ck))
    assert redo == [1]  # only the unfinished partition is rebuilt
    assert np.array_equal(resumed.adjacency, full.adjacency) and np.array_equal(resumed.degrees, full.degrees)
