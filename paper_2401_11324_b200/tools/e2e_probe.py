"""Break the end-to-end search time of one batch into its host/device parts
(diagnostic for bench.py's e2e number)."""

from __future__ import annotations

import ctypes
import sys
import time

import numpy as np


def main(config="C2", t=80, reps=5):
    import torch
    from paper_2401_11324_b200 import GraphSearcher, _lib
    from paper_2401_11324_b200.tools.bench_data import build_artifacts
    art = build_artifacts(config, cache_dir="/tmp/bang_bench_cache")
    s = GraphSearcher(k=10, t=t, mode="in_memory", batch_size=10_000)
    s.fit(art["base"], graph=art["graph"], codebook=art["codebook"], codes=art["codes"])
    qpin = torch.empty(art["queries"].shape, dtype=torch.float32, pin_memory=True)
    qpin.copy_(torch.from_numpy(art["queries"]))
    q = qpin.numpy()
    ix = s.index_
    L = _lib.lib()
    nq, k = q.shape[0], 10
    for _ in range(reps):
        bufs = [np.empty((nq, k), np.int32), np.empty((nq, k), np.float32), np.empty(nq, np.int32),
                np.empty(nq, np.uint8), np.empty(nq, np.uint8), np.empty(nq, np.float64),
                np.empty(nq + 1, np.int64)]
        t0 = time.perf_counter()
        st = L.bang_search(ix.handle, _lib.ptr(q), nq, k, t, 399_887, _lib.RERANK, *[_lib.ptr(b) for b in bufs],
                           None, 0)
        t1 = time.perf_counter()
        flat = np.empty(int(bufs[-1][-1]), np.int32)
        L.bang_last_visit_logs(ix.handle, _lib.ptr(flat), flat.size)
        t2 = time.perf_counter()
        res = s.search(q)
        t3 = time.perf_counter()
        stt = ix.stats()
        print(f"bang_search {1e3 * (t1 - t0):.3f} ms (kernel {stt['kernel_ms']:.3f} ms), "
              f"visit logs {1e3 * (t2 - t1):.3f} ms, full GraphSearcher.search {1e3 * (t3 - t2):.3f} ms", flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["C2"]), *(int(a) for a in sys.argv[2:3]))
