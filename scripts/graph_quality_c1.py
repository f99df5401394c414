"""Graph-builder quality check against the reference's own Vamana graph (C1).

Recall@10 / mean iterations of the oracle search at several t over
  (a) the reference VamanaBuilder(32, 64, 1.2) graph stored in
      tests/golden/c1_reference.npz, and
  (b) tools/graph_build.build_graph (+ search-based refine passes) on the
      same data, same codebook and codes.
Runs on the CPU (torch CPU for the builder, the C oracle for searches):
    python scripts/graph_quality_c1.py [--passes 2] [--refine-t 64]
Diagnostic for SURVEY.md 8(f) f3 only; nothing here is timed or shipped.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2401_11324_b200.tools.datasets import gaussian_mixture  # noqa: E402


def recall(ids, gt):
    return float(np.mean([len(set(a[a >= 0]) & set(b)) / gt.shape[1] for a, b in zip(ids, gt)]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--passes", type=int, default=2)
    ap.add_argument("--refine-t", type=int, default=64)
    ap.add_argument("--sigma", type=float, default=1.2)
    ap.add_argument("--ts", default="24,32,48,64")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    a = ap.parse_args()
    import torch
    torch.set_num_threads(a.threads)
    g = np.load(os.path.join(ROOT, "tests/golden/c1_reference.npz"))
    base, q = gaussian_mixture(100_000, 1_000, 128, clusters=1024, seed=0)
    xb = torch.from_numpy(base).double()
    xq = torch.from_numpy(q).double()
    d = (xq.square().sum(1)[:, None] + xb.square().sum(1)[None, :] - 2 * xq @ xb.T)
    gt = torch.topk(d, 10, dim=1, largest=False).indices.numpy()
    sizes = g["sub_sizes"]
    cents = np.split(g["centroids"], np.cumsum(sizes * 256)[:-1])
    cents = [c.reshape(256, s) for c, s in zip(cents, sizes)]
    ts = [int(v) for v in a.ts.split(",")]

    def evaluate(name, adj, deg, medoid):
        out = {}
        for t in ts:
            r = O.search(q, centroids=cents, sub_sizes=sizes, codes=g["codes"], adjacency=adj, degrees=deg,
                         medoid=medoid, vectors=base, k=10, t=t, bloom_entries=399_887, threads=a.threads)
            out[t] = (round(recall(r["ids"], gt), 4), round(float(r["iterations"].mean()), 1))
        print(f"{name:32s} " + "  ".join(f"t={t}: R@10 {v[0]:.4f} I {v[1]}" for t, v in out.items()), flush=True)
        return out

    evaluate("reference VamanaBuilder", g["adjacency"], g["degrees"], int(g["medoid"]))

    from paper_2401_11324_b200.tools import graph_build as GB
    t0 = time.time()
    gi = GB.build_graph(base, degree_bound=32, build_worklist=64, sigma=a.sigma, device="cpu")
    print(f"build {time.time() - t0:.1f}s (medoid {gi.medoid}, ref medoid {int(g['medoid'])})")
    evaluate("build_graph", gi.adjacency, gi.degrees, gi.medoid)
    x = torch.from_numpy(base)
    adj = torch.from_numpy(gi.adjacency).long()
    deg = torch.from_numpy(gi.degrees).long()
    for p in range(a.passes):
        A, D = adj.to(torch.int32).numpy(), deg.to(torch.int32).numpy()

        def visit_fn(lo, hi):
            r = O.search(base[lo:hi], centroids=cents, sub_sizes=sizes, codes=g["codes"], adjacency=A,
                         degrees=D, medoid=gi.medoid, vectors=base, k=10, t=a.refine_t,
                         bloom_entries=399_887, threads=a.threads)
            lens = np.array([len(v) for v in r["visit_logs"]], np.int64)
            offs = np.concatenate([[0], np.cumsum(lens)])
            return offs, np.concatenate(r["visit_logs"])

        t0 = time.time()
        adj, deg = GB.refine_graph(x, adj, deg, visit_fn, 32, a.sigma, chunk=1 << 20)
        adj = torch.where(torch.arange(32)[None, :] < deg[:, None], adj, torch.full_like(adj, -1))
        print(f"refine pass {p + 1}: {time.time() - t0:.1f}s")
        evaluate(f"build_graph + {p + 1} pass(es) t={a.refine_t}", adj.to(torch.int32).numpy(),
                 deg.to(torch.int32).numpy(), gi.medoid)


if __name__ == "__main__":
    main()
