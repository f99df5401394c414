"""Benchmark artifacts for the BASELINE.json configurations, built on the GPU.

(base, queries, graph, codebook, codes, ground truth) for a named config,
deterministic for a seed.  An optional on-disk cache only skips rebuilding
(the artifacts are identical either way); nothing is timed here.
"""

from __future__ import annotations

import hashlib
import os
import time

import numpy as np

from ..graph import GraphIndex
from ..pq import CompressedVectors, PQCodebook
from .datasets import gaussian_mixture, to_u8

CONFIGS = {
    # name: (n, nq, dim, dtype, clusters, R, m, description)
    "C1": (100_000, 1_000, 128, "f32", 1024, 32, 32,
           "synthetic 100Kx128 fp32 Gaussian-mixture, R=32, PQ 32x256, 1K queries, k=10"),
    "C2": (1_000_000, 10_000, 128, "u8", 10_000, 64, 32,
           "SIFT1M-shape synthetic 1Mx128 uint8, R=64, PQ 32 subspaces, 10K queries, k=10"),
    "C3": (10_000_000, 10_000, 96, "f32", 100_000, 64, 48,
           "DEEP-shape synthetic 10Mx96 fp32, R=64, PQ 48 subspaces, 10K queries, k=10"),
    # BASELINE.json configs[3] with a real graph: the graph and vectors live
    # in pinned host memory (mode="pipelined"); the graph is built in
    # overlapping partitions (PARTITIONED)
    "C4": (100_000_000, 10_000, 128, "u8", 1_000_000, 64, 32,
           "SIFT-shape synthetic 100Mx128 uint8, R=64, PQ 32 subspaces, graph + vectors in pinned host memory, "
           "10K queries, k=10"),
    # C4 with clusters half as wide (cluster_scale 0.5): at 100M points the
    # default-width mixture has almost no neighbourhood contrast (mean
    # d10/d100 = 0.78 already at 400K; recall@10 0.54 at t=256 on the real
    # partitioned graph, profiles/r02/c4/), unlike SIFT; at 0.5 it is 0.42
    "C4t": (100_000_000, 10_000, 128, "u8", 1_000_000, 64, 32,
            "SIFT-shape synthetic 100Mx128 uint8 (clusters half as wide), R=64, PQ 32 subspaces, graph + vectors "
            "in pinned host memory, 10K queries, k=10"),
    # reduced-n variants of the same shapes (parity tests, quick checks)
    "C2s": (100_000, 10_000, 128, "u8", 1_000, 64, 32, "C2 shape at n=100K"),
    "C3s": (200_000, 10_000, 96, "f32", 2_000, 64, 48, "C3 shape at n=200K"),
    "C3p": (10_000_000, 10_000, 96, "f32", 100_000, 64, 48, "C3 built by partitions (builder check)"),
}

# Configs whose graph is built in overlapping partitions
# (graph_build.build_graph_partitioned): parts, overlap, search-based passes
# per partition.  C4's monolithic build would need ~230 GB of HBM (k-NN
# candidate tables); C3p checks the partitioned build against C3's.
CLUSTER_SCALE = {"C4t": 0.5}
PARTITIONED = {
    "C4": dict(parts=24, overlap=2, refine=(128,)),
    "C4t": dict(parts=24, overlap=2, refine=(128,)),
    "C3p": dict(parts=4, overlap=2, refine=(128,)),
}
# Configs searched with the graph in pinned host memory (BASELINE.json configs[3])
HOST_GRAPH_CONFIGS = ("C4", "C4t")


# Throughput-only shapes (BASELINE.json configs[3..4]; "C5:
# seeded random 64-regular graph ... C5 has no recall").  The graph, codes,
# codebook and u8 vectors are seeded random; the graph and vectors live in
# pinned host memory (mode="pipelined").  C5's 1B x 64 adjacency (256 GB)
# exceeds a single box's host RAM, so its shape is run at the largest n that
# fits alongside C4.
THROUGHPUT_CONFIGS = {
    # name: (n, nq, dim, R, m, t, description)
    "C4r": (100_000_000, 10_000, 128, 64, 32, 80,
            "SIFT-shape 100Mx128 uint8, random 64-regular graph in pinned host memory "
            "(throughput only, no recall), PQ 32 subspaces in HBM, 10K queries, t=80"),
}

EXACT_KNN_LIMIT = 2_000_000
# search-based Vamana passes after the partitioned k-NN graph (n > EXACT_KNN_LIMIT):
# the worklist t of each pass.  At C3 two t=128 passes lift recall@10 at t=200
# from 0.846 to 0.911, a third at t=200 to 0.918 (0.897 at t=160)
# (profiles/r01/c3_graph_study*.jsonl).
REFINE = (128, 128, 200)
# Index layout of the real-graph configs: "partition" relabels the built index
# so graph neighbours are near in memory (graph_build.locality_order);
# "natural" (default) keeps the generator's order.  Measured at C3: no QPS
# difference (720K vs 726K, profiles/r01/layout_C3.txt) -- the search is bound
# by per-iteration latency, not by DRAM pages.  BANG_BENCH_LAYOUT overrides.
LAYOUT = os.environ.get("BANG_BENCH_LAYOUT", "natural")


def refine_with_search(base, graph, codebook, codes, R, t=64, sigma=1.2, chunk=1 << 20, log=print):
    """graph_build.refine_graph with visit logs from GraphSearcher (t=64)."""
    import torch
    from .._dev import torch_device
    from ..engine import GraphSearcher
    from .graph_build import refine_graph
    dev = torch_device()
    s = GraphSearcher(k=10, t=t, mode="in_memory", batch_size=chunk)
    s.fit(base, graph=graph, codebook=codebook, codes=codes)

    def visit_fn(lo, hi):
        return s.search(base[lo:hi]).visit_logs.csr()

    x = torch.from_numpy(np.ascontiguousarray(base, np.float32)).to(dev)
    adj = torch.from_numpy(graph.adjacency).to(dev).long()
    deg = torch.from_numpy(graph.degrees).to(dev).long()
    adj, deg = refine_graph(x, adj, deg, visit_fn, R, sigma, chunk=chunk, log=log)
    del s
    adj_np = adj.to(torch.int32).cpu().numpy()
    deg_np = deg.to(torch.int32).cpu().numpy()
    adj_np[np.arange(R)[None, :] >= deg_np[:, None]] = -1
    return GraphIndex(adj_np, deg_np, graph.medoid, R, validate=False)


def build_random_artifacts(name: str, seed: int = 0, nq_total: int | None = None, log=print):
    """Seeded random index of a throughput-only shape (no ground truth)."""
    import torch
    from .._dev import torch_device
    n, nq, dim, R, m, t, desc = THROUGHPUT_CONFIGS[name]
    nq_total = nq_total or nq
    dev = torch_device()
    g = torch.Generator(device=dev).manual_seed(seed)
    t0 = time.time()
    chunk = 1 << 24
    adj = np.empty((n, R), np.int32)
    vec = np.empty((n, dim), np.uint8)
    codes = np.empty((n, m), np.uint8)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        a = torch.randint(0, n - 1, (hi - lo, R), generator=g, device=dev, dtype=torch.int64)
        own = torch.arange(lo, hi, device=dev)[:, None]
        a = torch.where(a >= own, a + 1, a)  # uniform over the other n-1 nodes: no self-loops
        adj[lo:hi] = a.to(torch.int32).cpu().numpy()
        vec[lo:hi] = torch.randint(0, 256, (hi - lo, dim), generator=g, device=dev, dtype=torch.int32).to(
            torch.uint8).cpu().numpy()
        codes[lo:hi] = torch.randint(0, 256, (hi - lo, m), generator=g, device=dev, dtype=torch.int32).to(
            torch.uint8).cpu().numpy()
    deg = np.full(n, R, np.int32)
    queries = torch.randint(0, 256, (nq_total, dim), generator=g, device=dev, dtype=torch.int32).float().cpu().numpy()
    sub = dim // m
    cents = [torch.randint(0, 256, (256, sub), generator=g, device=dev, dtype=torch.int32).float().cpu().numpy()
             for _ in range(m)]
    # medoid: the point nearest the mean of a 1M-point sample (graph.py:107-115 on a sample)
    samp = torch.from_numpy(vec[:: max(1, n // 1_000_000)]).to(dev).double()
    medoid = int(((samp - samp.mean(0)) ** 2).sum(1).argmin().item()) * max(1, n // 1_000_000)
    log(f"[bench_data] {name}: random artifacts in {time.time() - t0:.1f}s")
    return dict(base=vec, queries=queries,
                graph=GraphIndex(adj, deg, medoid, R, validate=False),
                codebook=PQCodebook(dim=dim, subspace_sizes=[sub] * m, centroids=cents),
                codes=CompressedVectors(codes), gt_ids=None, gt_dists=None,
                meta=dict(desc=desc, n=n, dim=dim, dtype="u8", R=R, m=m, clusters=0, t=t,
                          throughput_only=True))


def _key(name, seed, nq_total):
    return hashlib.sha1(f"v3|{name}|{CONFIGS[name]}|{REFINE}|{seed}|{nq_total}|{LAYOUT}".encode()).hexdigest()[:16]


_ARRAYS = ("base", "queries", "adjacency", "degrees", "medoid", "sub_sizes", "centroids", "codes",
           "gt_ids", "gt_dists")


def cache_path(name: str, seed: int, nq_total: int, cache_dir: str) -> str:
    return os.path.join(cache_dir, f"bang_{name}_{_key(name, seed, nq_total)}")


def _load_cached(path, name, meta, log):
    """Arrays are memory-mapped .npy files: ranks on one box share the page cache."""
    d = {k: np.load(os.path.join(path, k + ".npy"), mmap_mode="r") for k in _ARRAYS}
    R = meta["R"]
    sizes = [int(s) for s in d["sub_sizes"]]
    cents, pos = [], 0
    cat = np.asarray(d["centroids"])
    for s in sizes:
        cents.append(cat[pos:pos + 256 * s].reshape(256, s))
        pos += 256 * s
    log(f"[bench_data] {name}: loaded cached artifacts {path}")
    return dict(base=d["base"], queries=np.asarray(d["queries"]),
                graph=GraphIndex(d["adjacency"], np.asarray(d["degrees"]), int(d["medoid"]), R, validate=False),
                codebook=PQCodebook(dim=meta["dim"], subspace_sizes=sizes, centroids=cents),
                codes=CompressedVectors(d["codes"]), gt_ids=np.asarray(d["gt_ids"]),
                gt_dists=np.asarray(d["gt_dists"]), meta=meta)


def _save_cached(path, arrays, log):
    tmp = path + ".tmp"
    try:
        os.makedirs(tmp, exist_ok=True)
        for k in _ARRAYS:
            np.save(os.path.join(tmp, k + ".npy"), np.asarray(arrays[k]))
        os.replace(tmp, path)
    except OSError as e:  # a full scratch disk only costs the cache
        log(f"[bench_data] cache not written ({e})")
        import shutil
        shutil.rmtree(tmp, ignore_errors=True)


def _ck_has(ck, *names) -> bool:
    return all(os.path.exists(os.path.join(ck, k + ".npy")) for k in names)


def _ck_load(ck, name):
    return np.load(os.path.join(ck, name + ".npy"), mmap_mode="r")


def _ck_save(ck, **arrays) -> None:
    """Each array written to a temporary name, then renamed: a checkpoint
    file is complete or absent."""
    for k, a in arrays.items():
        tmp = os.path.join(ck, k + ".tmp.npy")
        np.save(tmp, np.asarray(a))
        os.replace(tmp, os.path.join(ck, k + ".npy"))


def build_artifacts(name: str, seed: int = 0, nq_total: int | None = None, cache_dir: str | None = None,
                    log=print, load_only: bool = False):
    """Returns dict(base, queries, graph, codebook, codes, gt_ids, gt_dists, meta).
    load_only: the caller knows another process has written the cache."""
    from .graph_build import build_graph
    from .groundtruth import brute_force_knn
    from .pq_train import encode, train_codebook

    if name in THROUGHPUT_CONFIGS:
        return build_random_artifacts(name, seed, nq_total, log)
    n, nq, dim, dt, clusters, R, m, desc = CONFIGS[name]
    nq_total = nq_total or nq
    meta = dict(desc=desc, n=n, dim=dim, dtype=dt, R=R, m=m, clusters=clusters, layout=LAYOUT)
    path = None
    if cache_dir:
        os.makedirs(cache_dir, exist_ok=True)
        path = cache_path(name, seed, nq_total, cache_dir)
        if os.path.isdir(path) or load_only:
            return _load_cached(path, name, meta, log)
    t0 = time.time()
    # the partitioned (C4-size) builds checkpoint every stage to disk so a
    # build longer than one GPU session resumes where it stopped
    ck = None
    if name in PARTITIONED:
        ck = os.path.join(cache_dir or "/tmp", f"bang_{name}_ckpt_{_key(name, seed, nq_total)}")
        os.makedirs(ck, exist_ok=True)
    if ck and _ck_has(ck, "base", "queries"):
        base, queries = _ck_load(ck, "base"), np.asarray(_ck_load(ck, "queries"))
        log(f"[bench_data] {name}: data from checkpoint {ck}")
    else:
        base, queries = gaussian_mixture(n, nq_total, dim, clusters=clusters, seed=seed,
                                         cluster_scale=CLUSTER_SCALE.get(name, 1.0),
                                         out_dtype=np.uint8 if dt == "u8" else np.float32)
        if dt == "u8":
            queries = queries.astype(np.float32)
        if ck:
            _ck_save(ck, base=base, queries=queries)
    t1 = time.time()
    if name in PARTITIONED:
        from .graph_build import build_graph_partitioned
        if _ck_has(ck, "centroids", "sub_sizes", "codes"):
            cat, sizes = np.asarray(_ck_load(ck, "centroids")), [int(v) for v in _ck_load(ck, "sub_sizes")]
            cents, pos = [], 0
            for sz in sizes:
                cents.append(cat[pos:pos + 256 * sz].reshape(256, sz))
                pos += 256 * sz
            cb = PQCodebook(dim=dim, subspace_sizes=sizes, centroids=cents)
            codes = CompressedVectors(np.asarray(_ck_load(ck, "codes")))
        else:
            cb = train_codebook(base, m=m, iters=15, seed=seed)
            codes = encode(base, cb)
            _ck_save(ck, centroids=cb.concatenated(), sub_sizes=np.asarray(cb.subspace_sizes, np.int32),
                     codes=codes.codes)
        t2 = time.time()
        cfg = PARTITIONED[name]

        def refine_fn(members, g, t_ref):
            return refine_with_search(base[members], g, cb, CompressedVectors(codes.codes[members]), R,
                                      t=t_ref, log=log)

        if _ck_has(ck, "adjacency", "degrees", "medoid"):
            graph = GraphIndex(_ck_load(ck, "adjacency"), np.asarray(_ck_load(ck, "degrees")),
                               int(_ck_load(ck, "medoid")), R, validate=False)
        else:
            # the per-partition checkpoint (an (n, overlap*R) int32 table,
            # 51 GB at C4) only where the scratch disk holds it
            import shutil
            cand_bytes = n * cfg["overlap"] * R * 4
            part_ck = ck if shutil.disk_usage(ck).free > 1.5 * cand_bytes + 32 * n else None
            graph = build_graph_partitioned(base, degree_bound=R, parts=cfg["parts"], overlap=cfg["overlap"],
                                            refine_fn=refine_fn, refine=cfg["refine"], seed=seed, log=log,
                                            ckpt_dir=part_ck)
            _ck_save(ck, adjacency=graph.adjacency, degrees=graph.degrees, medoid=np.int64(graph.medoid))
        t3 = time.time()
        t2, t3 = t3 - (t2 - t1), t3  # report graph time apart from PQ time
    else:
        graph = build_graph(base, degree_bound=R, seed=seed, log=log)
        t2 = time.time()
        cb = train_codebook(base, m=m, iters=15, seed=seed)
        codes = encode(base, cb)
        t3 = time.time()
    if n > EXACT_KNN_LIMIT and name not in PARTITIONED:
        # partitioned k-NN graph -> one search-based Vamana pass with the
        # B200 search itself (the reference's builder, graph.py:251-344,
        # inserts by greedy search too)
        for t_ref in REFINE:
            graph = refine_with_search(base, graph, cb, codes, R, t=t_ref, log=log)
        t2 += time.time() - t3
        t3 = time.time()
    if LAYOUT == "partition":
        from .graph_build import locality_order, relabel_index
        perm = locality_order(base, seed=seed)
        base, adj, deg, med = relabel_index(perm, base, graph.adjacency, graph.degrees, graph.medoid)
        graph = GraphIndex(adj, deg, med, R, validate=False)
        codes = CompressedVectors(np.ascontiguousarray(codes.codes[perm]))
        log(f"[bench_data] {name}: relabelled in k-means partition order ({time.time() - t3:.1f}s)")
    if ck and _ck_has(ck, "gt_ids", "gt_dists"):
        gt_ids, gt_d = np.asarray(_ck_load(ck, "gt_ids")), np.asarray(_ck_load(ck, "gt_dists"))
    else:
        gt_ids, gt_d = brute_force_knn(base, queries, 10)
        if ck:
            _ck_save(ck, gt_ids=gt_ids, gt_dists=gt_d)
    t4 = time.time()
    log(f"[bench_data] {name}: data {t1 - t0:.1f}s graph {t2 - t1:.1f}s pq {t3 - t2:.1f}s gt {t4 - t3:.1f}s"
        f" (mean degree {graph.degrees.mean():.1f})")
    if path:
        _save_cached(path, dict(base=base, queries=queries, adjacency=graph.adjacency, degrees=graph.degrees,
                                medoid=np.int64(graph.medoid),
                                sub_sizes=np.asarray(cb.subspace_sizes, np.int32),
                                centroids=cb.concatenated(), codes=codes.codes, gt_ids=gt_ids,
                                gt_dists=gt_d), log)
    return dict(base=base, queries=queries, graph=graph, codebook=cb, codes=codes, gt_ids=gt_ids,
                gt_dists=gt_d, meta=meta)
