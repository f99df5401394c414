"""Multi-GPU host logic: contiguous query shards, in-order
host gather, world_size-2 process groups over gloo on CPU.

The per-shard search here is the pinned CPU oracle (the checker, standing in
for one GPU's bang_search); the GPU test at the bottom runs the real
ShardedSearcher on every visible device.
"""

import os

import numpy as np
import pytest

import golden_util as gu
from oracle import oracle as O
from paper_2401_11324_b200.engine import SearchResult, VisitLogs
from paper_2401_11324_b200.errors import ParameterError
from paper_2401_11324_b200.sharding import distributed_search, merge_results, shard_range

CASE = "search_vamana_r40_uneven.npz"


@pytest.mark.parametrize("nq,world", [(0, 2), (1, 2), (7, 2), (10_000, 8), (10_001, 8), (3, 8), (40, 3)])
def test_shard_ranges_partition_the_batch(nq, world):
    rs = [shard_range(nq, world, r) for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == nq
    for (a, b), (c, d) in zip(rs, rs[1:]):
        assert b == c and a <= b and c <= d
    per = -(-nq // world)
    assert all(hi - lo <= per for lo, hi in rs)


def test_shard_range_rejects_bad_rank():
    with pytest.raises(ParameterError):
        shard_range(10, 2, 2)
    with pytest.raises(ParameterError):
        shard_range(10, 0, 0)


def _oracle_search_fn(g):
    cents = gu.split_centroids(g["centroids"], g["sub_sizes"])

    def run(q):
        out = O.search(q, centroids=cents, sub_sizes=g["sub_sizes"], codes=g["codes"],
                       adjacency=g["adjacency"], degrees=g["degrees"], medoid=int(g["medoid"]),
                       vectors=g["base"], k=int(g["k"]), t=int(g["t"]),
                       bloom_entries=int(g["bloom_entries"]), rerank=bool(g["rerank"]))
        n = q.shape[0]
        return SearchResult(ids=out["ids"], dists=out["dists"], iterations=out["iterations"],
                            converged=out["converged"], wall_times=np.zeros(n), elapsed=0.0,
                            short=out["short"], visit_logs=VisitLogs.concat([out["visit_logs"]]))
    return run


def _assert_matches_golden(res, g):
    assert np.array_equal(res.ids, g["ids"])
    assert np.array_equal(res.dists, g["dists"])
    assert np.array_equal(res.iterations, g["iterations"])
    want = gu.logs(g["log_offsets"], g["log_ids"])
    assert len(res.visit_logs) == len(want)
    for a, b in zip(res.visit_logs, want):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_merged_shards_equal_the_reference_batch(world):
    g = gu.load(CASE)
    run = _oracle_search_fn(g)
    q = g["queries"]
    parts = [run(q[slice(*shard_range(q.shape[0], world, r))]) for r in range(world)]
    _assert_matches_golden(merge_results(parts), g)


def test_visit_logs_concat_keeps_query_order():
    a = VisitLogs.concat([[np.array([1, 2]), np.array([3])]])
    b = VisitLogs.concat([[np.array([], np.int64)], a])
    assert len(b) == 3
    assert [list(x) for x in b] == [[], [1, 2], [3]]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = gu.load(CASE)
        res = distributed_search(_oracle_search_fn(g), g["queries"])
        _assert_matches_golden(res, g)
        # every rank searched only its own shard
        lo, hi = shard_range(g["queries"].shape[0], world, rank)
        q.put((rank, lo, hi, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, -1, -1, repr(e)))
    finally:
        dist.destroy_process_group()


def test_distributed_search_gloo_world2():
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [o[3] for o in out] == ["ok", "ok"], out
    assert out[0][1] == 0 and out[0][2] == out[1][1] and out[1][2] == gu.load(CASE)["queries"].shape[0]


@pytest.mark.gpu
def test_sharded_searcher_on_all_visible_gpus_matches_reference():
    import torch

    import paper_2401_11324_b200 as B
    from paper_2401_11324_b200.sharding import ShardedSearcher
    g = gu.load(CASE)
    cents = gu.split_centroids(g["centroids"], g["sub_sizes"])
    cb = B.PQCodebook(dim=g["base"].shape[1], subspace_sizes=[int(s) for s in g["sub_sizes"]],
                      centroids=cents)
    graph = B.GraphIndex(g["adjacency"], g["degrees"], int(g["medoid"]), int(g["degree_bound"]))
    # one replica per visible GPU; on a 1-GPU box two replicas share device 0
    devs = list(range(torch.cuda.device_count())) or [0]
    if len(devs) == 1:
        devs = [0, 0]
    ss = ShardedSearcher(devs, k=int(g["k"]), t=int(g["t"]), mode="in_memory",
                         bloom_entries=int(g["bloom_entries"]), rerank=bool(g["rerank"]))
    try:
        ss.fit(g["base"], graph=graph, codebook=cb, codes=B.CompressedVectors(g["codes"]))
        _assert_matches_golden(ss.search(g["queries"]), g)
    finally:
        ss.close()
