"""Debug: the smoke's C3-shaped random index (numpy only), split kernel,
compared with the oracle; run under an outer `timeout`."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O
import paper_2401_11324_b200 as B
nq = int(sys.argv[1]); t = int(sys.argv[2]); opts = dict(kv.split("=") for kv in sys.argv[3:])
rng = np.random.default_rng(11)
n, d, R, m = 4_000, 96, 64, 48
base = rng.normal(size=(n, d)).astype(np.float32)
q = rng.normal(size=(nq, d)).astype(np.float32)
adj = np.empty((n, R), np.int32)
for i in range(n):
    adj[i] = (i + 1 + rng.choice(n - 1, size=R, replace=False)) % n
deg = np.full(n, R, np.int32)
cents = [rng.normal(size=(256, 2)).astype(np.float32) for _ in range(m)]
codes = rng.integers(0, 256, size=(n, m), dtype=np.uint8)
cb = B.PQCodebook(dim=d, subspace_sizes=[2] * m, centroids=cents)
s = B.GraphSearcher(k=10, t=t, mode="in_memory", debug_checks=True)
s.fit(base, graph=B.GraphIndex(adj, deg, 0, R), codebook=cb, codes=B.CompressedVectors(codes))
s.set_kernel(opts.pop("kernel", "split"), **{k: int(v) for k, v in opts.items()})
print("searching", flush=True)
res = s.search(q)
want = O.search(q, centroids=cents, sub_sizes=[2] * m, codes=codes, adjacency=adj, degrees=deg, medoid=0,
                vectors=base, k=10, t=t, bloom_entries=399_887)
ok = np.array_equal(res.ids, want["ids"]) and np.array_equal(res.iterations, want["iterations"])
print("nq", nq, "t", t, "ok" if ok else "MISMATCH", s.last_stats()["kernel"], res.iterations[:6], want["iterations"][:6], flush=True)
