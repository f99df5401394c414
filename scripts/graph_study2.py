"""C3 graph-quality study (offline tooling).

Starts from the benchmark's own C3 graph (bench_data.build_artifacts) and
applies further search-based Vamana passes, printing recall@10 and mean
iterations at several t after each stage; then rebuilds the base graph with a
wider IVF probe (better k-NN candidates) and repeats the pass schedule.

    python scripts/graph_study2.py [--stages 200:1.2,200:1.2,256:1.3] [--nprobe 24]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stages", default="200:1.2,200:1.2,256:1.2")
    ap.add_argument("--ts", default="64,100,128,166")
    ap.add_argument("--nprobe", type=int, default=24)
    ap.add_argument("--rebuild", default="128:1.2,128:1.2,200:1.2")
    ap.add_argument("--cache", default="/tmp/bang_bench_cache")
    args = ap.parse_args()
    import torch
    from paper_2401_11324_b200 import GraphIndex, GraphSearcher
    from paper_2401_11324_b200.tools import bench_data as bd
    from paper_2401_11324_b200.tools import graph_build as GB
    from paper_2401_11324_b200.tools.groundtruth import recall_at_k
    log = lambda *a: print(*a, file=sys.stderr, flush=True)
    art = bd.build_artifacts("C3", seed=0, cache_dir=args.cache, log=log)
    R = art["meta"]["R"]
    ts = [int(x) for x in args.ts.split(",")]

    def evaluate(graph, tag):
        out = {"graph": tag}
        s = GraphSearcher(k=10, t=max(ts), mode="in_memory", batch_size=10_000)
        s.fit(art["base"], graph=graph, codebook=art["codebook"], codes=art["codes"])
        for t in ts:
            s.t = t
            r = s.search(art["queries"])
            out[f"t{t}"] = (round(recall_at_k(r.ids, art["gt_ids"], 10), 4), round(float(r.iterations.mean()), 1))
        del s
        print(json.dumps(out), flush=True)

    def passes(g, spec, tag):
        for i, st in enumerate(spec.split(",")):
            t_ref, sig = st.split(":")
            t0 = time.time()
            g = bd.refine_with_search(art["base"], g, art["codebook"], art["codes"], R, t=int(t_ref),
                                      sigma=float(sig), log=log)
            log(f"{tag} pass {i + 1} (t={t_ref}, sigma={sig}): {time.time() - t0:.1f}s")
            torch.cuda.empty_cache()
            evaluate(g, f"{tag} + pass t={t_ref} sigma={sig}")
        return g

    g = GraphIndex(np.asarray(art["graph"].adjacency), np.asarray(art["graph"].degrees), art["graph"].medoid, R,
                   validate=False)
    evaluate(g, "bench graph")
    passes(g, args.stages, "bench graph")

    # wider IVF probe for the initial k-NN candidates, then the bench schedule
    dev = torch.device("cuda")
    x = torch.from_numpy(np.ascontiguousarray(art["base"], dtype=np.float32)).to(dev)
    t0 = time.time()
    ids, d = GB.knn_ivf(x, 2 * R, nprobe=args.nprobe)
    ids, d = GB._sort_rows_by_dist(ids, d)
    ids = torch.where(torch.isinf(d), torch.full_like(ids, -1), ids)
    adj, deg = GB.robust_prune(x, ids, d, R, 1.2)
    del ids, d
    adj, deg = GB.add_reverse_edges(x, adj, deg, R, 1.2)
    log(f"nprobe={args.nprobe} base graph: {time.time() - t0:.1f}s")
    adj_np = adj.to(torch.int32).cpu().numpy()
    deg_np = deg.to(torch.int32).cpu().numpy()
    adj_np[np.arange(R)[None, :] >= deg_np[:, None]] = -1
    del x, adj, deg
    torch.cuda.empty_cache()
    g2 = GraphIndex(adj_np, deg_np, art["graph"].medoid, R, validate=False)
    evaluate(g2, f"knn nprobe={args.nprobe}")
    passes(g2, args.rebuild + "," + args.stages, f"nprobe={args.nprobe}")


if __name__ == "__main__":
    main()
