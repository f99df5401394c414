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
    # reduced-n variants of the same shapes (parity tests, quick checks)
    "C2s": (100_000, 10_000, 128, "u8", 1_000, 64, 32, "C2 shape at n=100K"),
    "C3s": (200_000, 10_000, 96, "f32", 2_000, 64, 48, "C3 shape at n=200K"),
}


def _key(name, seed, nq_total):
    return hashlib.sha1(f"v2|{name}|{CONFIGS[name]}|{seed}|{nq_total}".encode()).hexdigest()[:16]


def build_artifacts(name: str, seed: int = 0, nq_total: int | None = None, cache_dir: str | None = None,
                    log=print):
    """Returns dict(base, queries, graph, codebook, codes, gt_ids, gt_dists, meta)."""
    from .graph_build import build_graph
    from .groundtruth import brute_force_knn
    from .pq_train import encode, train_codebook

    n, nq, dim, dt, clusters, R, m, desc = CONFIGS[name]
    nq_total = nq_total or nq
    path = None
    if cache_dir:
        os.makedirs(cache_dir, exist_ok=True)
        path = os.path.join(cache_dir, f"bang_{name}_{_key(name, seed, nq_total)}.npz")
        if os.path.exists(path):
            with np.load(path) as z:
                d = {k: z[k] for k in z.files}
            sizes = [int(s) for s in d["sub_sizes"]]
            cents, pos = [], 0
            for s in sizes:
                cents.append(d["centroids"][pos:pos + 256 * s].reshape(256, s))
                pos += 256 * s
            log(f"[bench_data] {name}: loaded cached artifacts {path}")
            return dict(base=d["base"], queries=d["queries"],
                        graph=GraphIndex(d["adjacency"], d["degrees"], int(d["medoid"]), R, validate=False),
                        codebook=PQCodebook(dim=dim, subspace_sizes=sizes, centroids=cents),
                        codes=CompressedVectors(d["codes"]), gt_ids=d["gt_ids"], gt_dists=d["gt_dists"],
                        meta=dict(desc=desc, n=n, dim=dim, dtype=dt, R=R, m=m, clusters=clusters))
    t0 = time.time()
    base, queries = gaussian_mixture(n, nq_total, dim, clusters=clusters, seed=seed)
    if dt == "u8":
        base, queries = to_u8(base), to_u8(queries).astype(np.float32)
    t1 = time.time()
    graph = build_graph(base, degree_bound=R, seed=seed)
    t2 = time.time()
    cb = train_codebook(base, m=m, iters=15, seed=seed)
    codes = encode(base, cb)
    t3 = time.time()
    gt_ids, gt_d = brute_force_knn(base, queries, 10)
    t4 = time.time()
    log(f"[bench_data] {name}: data {t1 - t0:.1f}s graph {t2 - t1:.1f}s pq {t3 - t2:.1f}s gt {t4 - t3:.1f}s"
        f" (mean degree {graph.degrees.mean():.1f})")
    if path:
        tmp = path + ".tmp.npz"
        np.savez(tmp, base=base, queries=queries, adjacency=graph.adjacency, degrees=graph.degrees,
                 medoid=np.int64(graph.medoid), sub_sizes=np.asarray(cb.subspace_sizes, np.int32),
                 centroids=cb.concatenated(), codes=codes.codes, gt_ids=gt_ids, gt_dists=gt_d)
        os.replace(tmp, path)
    return dict(base=base, queries=queries, graph=graph, codebook=cb, codes=codes, gt_ids=gt_ids,
                gt_dists=gt_d, meta=dict(desc=desc, n=n, dim=dim, dtype=dt, R=R, m=m, clusters=clusters))
