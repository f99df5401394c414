"""Graph-quality study for the large configs (offline tooling, not the hot path).

Builds a config's artifacts, then alternates search-based Vamana refinement
passes with recall checks in both PQ and exact-distance traversal, so the
graph's share of a recall shortfall is separated from PQ's.

    python scripts/graph_study.py --config C3 --passes 2 --refine-t 128
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
    ap.add_argument("--config", default="C3")
    ap.add_argument("--passes", type=int, default=2)
    ap.add_argument("--refine-t", type=int, default=128)
    ap.add_argument("--ts", default="64,128,200")
    ap.add_argument("--sigma", type=float, default=1.2)
    ap.add_argument("--modes", default="in_memory,exact_distance")
    args = ap.parse_args()
    import torch
    from paper_2401_11324_b200 import GraphSearcher
    from paper_2401_11324_b200.tools import bench_data as bd
    from paper_2401_11324_b200.tools.groundtruth import recall_at_k
    log = lambda *a: print(*a, file=sys.stderr, flush=True)
    art = bd.build_artifacts(args.config, seed=0, cache_dir=None, log=log)
    R = art["meta"]["R"]
    ts = [int(x) for x in args.ts.split(",")]

    def evaluate(graph, tag):
        out = {"graph": tag}
        for mode in args.modes.split(","):
            s = GraphSearcher(k=10, t=max(ts), mode=mode, batch_size=10_000)
            s.fit(art["base"], graph=graph, codebook=art["codebook"], codes=art["codes"])
            for t in ts:
                s.t = t
                r = s.search(art["queries"])
                out[f"{mode}_t{t}"] = (round(recall_at_k(r.ids, art["gt_ids"], 10), 4),
                                       round(float(r.iterations.mean()), 1))
            del s
        print(json.dumps(out), flush=True)

    g = art["graph"]
    evaluate(g, "built")
    for p in range(args.passes):
        t0 = time.time()
        g = bd.refine_with_search(art["base"], g, art["codebook"], art["codes"], R, t=args.refine_t,
                                  sigma=args.sigma, log=log)
        log(f"pass {p + 1}: {time.time() - t0:.1f}s")
        torch.cuda.empty_cache()
        evaluate(g, f"+{p + 1} pass(es) t={args.refine_t} sigma={args.sigma}")


if __name__ == "__main__":
    main()
