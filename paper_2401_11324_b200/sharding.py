"""Query sharding across the GPUs of one box.

Every piece of per-query state (distance table, Bloom filter, worklist,
visit log) is private to its query and results do not depend on how a batch
is split (the reference pins this: tests/test_engine.py:122-134),
so multi-GPU search is pure partitioning:

* GPU g owns the contiguous query range ``shard_range(nq, G, g)``;
* the index (codes, codebook, graph, re-rank vectors) is replicated on
  every GPU -- one ``bang_index`` handle per device;
* results come back to the host per GPU and are concatenated in query
  order, mirroring the batch loop of engine.py:431-452.

There is no collective on the search path.  Two drivers:

``ShardedSearcher``      one process, one host thread per GPU (ctypes
                         releases the GIL for the whole bang_search call, so
                         the G searches run concurrently);
``distributed_search``   one process per GPU (torchrun): each rank searches
                         its own shard; the host-side gather of the result
                         objects uses the process group only after the
                         search (any backend, gloo on CPU in the tests).
"""

from __future__ import annotations

import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .engine import GraphSearcher, SearchResult, VisitLogs
from .errors import ParameterError


def shard_range(nq: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of rank's contiguous shard: ceil(nq/world) queries per rank,
    the last ranks possibly short or empty."""
    if world < 1 or not 0 <= rank < world:
        raise ParameterError(f"rank {rank} outside world of size {world}")
    per = -(-int(nq) // world)
    lo = min(int(nq), rank * per)
    return lo, min(int(nq), lo + per)


def merge_results(parts: list[SearchResult], elapsed: float | None = None) -> SearchResult:
    """Concatenate per-shard results in shard order (engine.py:444-452).
    ``elapsed`` defaults to the slowest shard's (shards run concurrently)."""
    parts = list(parts)
    if not parts:
        raise ParameterError("no shard results to merge")
    k = parts[0].ids.shape[1]
    if any(p.ids.shape[1] != k for p in parts):
        raise ParameterError("shards disagree on k")
    logs = VisitLogs.concat([p.visit_logs for p in parts])
    return SearchResult(
        ids=np.concatenate([p.ids for p in parts]),
        dists=np.concatenate([p.dists for p in parts]),
        iterations=np.concatenate([p.iterations for p in parts]),
        converged=np.concatenate([p.converged for p in parts]),
        wall_times=np.concatenate([p.wall_times for p in parts]),
        elapsed=max(p.elapsed for p in parts) if elapsed is None else float(elapsed),
        short=np.concatenate([p.short for p in parts]),
        visit_logs=logs)


class ShardedSearcher:
    """``GraphSearcher`` replicated on several GPUs of this process.

    ``ShardedSearcher(devices=[0, 1, ...], k=10, t=..., ...)`` takes the
    GraphSearcher parameters; ``fit`` uploads the same artifacts to every
    device, ``search`` splits the batch into contiguous per-device shards,
    searches them concurrently (one host thread per device) and returns one
    ``SearchResult`` equal to a single-GPU search of the whole batch.
    """

    def __init__(self, devices, **params):
        self.devices = [int(d) for d in devices]
        if not self.devices:
            raise ParameterError("at least one device is required")
        self.params = dict(params)
        self.searchers = [GraphSearcher(**self.params) for _ in self.devices]
        for s, d in zip(self.searchers, self.devices):
            s.device = d
        self._pool = ThreadPoolExecutor(max_workers=len(self.devices))

    def fit(self, X, y=None, graph=None, codebook=None, codes=None) -> "ShardedSearcher":
        # Missing artifacts are built ONCE (on this process's device) and the
        # same objects go to every replica: the builders' GPU reductions are
        # not bitwise deterministic, so per-replica builds could differ and
        # break the equal-to-one-GPU guarantee.
        data = getattr(X, "data", X)
        p = self.params
        if graph is None:
            from .tools.graph_build import build_graph
            graph = build_graph(np.asarray(data), degree_bound=p.get("degree_bound", 64),
                                build_worklist=p.get("build_worklist", 200), sigma=p.get("sigma", 1.2),
                                seed=p.get("seed", 0))
        if p.get("mode", "pipelined") != "exact_distance":
            if codebook is None:
                from .tools.pq_train import train_codebook
                codebook = train_codebook(np.asarray(data), m=p.get("m", 74), iters=p.get("pq_iters", 25),
                                          seed=p.get("seed", 0))
            if codes is None:
                from .tools.pq_train import encode
                codes = encode(np.asarray(data), codebook)
        # uploads are independent per device: run them concurrently
        futs = [self._pool.submit(s.fit, X, y, graph, codebook, codes) for s in self.searchers]
        for f in futs:
            f.result()
        return self

    def set_adc_variant(self, name: str) -> "ShardedSearcher":
        for s in self.searchers:
            s.set_adc_variant(name)
        return self

    def set_kernel(self, kernel: str = "auto", **tuning) -> "ShardedSearcher":
        for s in self.searchers:
            s.set_kernel(kernel, **tuning)
        return self

    def set_params(self, **params) -> "ShardedSearcher":
        """Search-time parameters (t, k, rerank, bloom_entries, ...) on every replica."""
        for s in self.searchers:
            s.set_params(**params)
        self.params.update(params)
        return self

    def search(self, queries, k: int | None = None) -> SearchResult:
        q = np.asarray(getattr(queries, "data", queries))
        nq = q.shape[0]
        G = len(self.devices)
        t0 = time.perf_counter()
        futs = []
        for g, s in enumerate(self.searchers):
            lo, hi = shard_range(nq, G, g)
            futs.append(self._pool.submit(s.search, q[lo:hi], k))
        parts = [f.result() for f in futs]
        return merge_results(parts, elapsed=time.perf_counter() - t0)

    def kneighbors(self, queries, n_neighbors: int | None = None, return_distance: bool = True):
        res = self.search(queries, k=n_neighbors)
        return (res.dists, res.ids) if return_distance else res.ids

    def close(self):
        for s in self.searchers:
            idx = getattr(s, "index_", None)
            if idx is not None:
                idx.close()
        self._pool.shutdown(wait=True)


def distributed_search(search_fn, queries, group=None) -> SearchResult:
    """One process per GPU: this rank searches ``shard_range(nq, world,
    rank)`` of ``queries`` with ``search_fn`` (e.g. a fitted GraphSearcher's
    ``search``), then every rank receives the merged result.  The gather is
    host-side object exchange over the process group AFTER the search; the
    search itself involves no communication."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    q = np.asarray(getattr(queries, "data", queries))
    lo, hi = shard_range(q.shape[0], world, rank)
    part = search_fn(q[lo:hi])
    parts = [None] * world
    dist.all_gather_object(parts, part, group=group)
    return merge_results(parts)
