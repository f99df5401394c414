"""Pin BASELINE config C1 against the READ-ONLY reference itself.

Run here (never on the GPU box -- /root/reference does not exist there):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_c1.py

BASELINE.json configs[0]: synthetic 100K x 128 f32 Gaussian mixture, Vamana
R=32 L=64, PQ 32 x 256, 1K queries, k=10.  Every artifact is made with the
reference's own code:
  data      bang.datasets.gaussian_mixture(100_000, 1_000, 128, clusters=1024,
            seed=0)                                    datasets.py:12-44
  graph     bang.graph.VamanaBuilder(32, 64, 1.2, seed=0)   graph.py:347-395
  codebook  bang.pq.ProductQuantizer(m=32, iters=25, seed=0) pq.py:185-235
  codes     bang.pq.compress_with_codebook                 pq.py:252-264
  outputs   bang.GraphSearcher(k=10, t, mode="in_memory", debug_checks=True)
            .search(queries) for t in (48, 152)           engine.py:409-452
The base vectors are NOT stored (51 MB): the repo's generator reproduces the
reference stream bit for bit, and the fixture keeps the SHA-256 of the base and
query bytes so the test proves it.  Everything else (graph, codebook, codes,
queries, ids, dists, iterations, visit logs) is stored.  The reference's own
QPS on this container's cores is recorded beside the outputs.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, REF_SRC)

import bang  # noqa: E402
from bang.datasets import gaussian_mixture  # noqa: E402
from bang.graph import VamanaBuilder  # noqa: E402
from bang.pq import ProductQuantizer, compress_with_codebook  # noqa: E402

T_VALUES = (48, 152)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    t0 = time.time()
    base, queries = gaussian_mixture(100_000, 1_000, 128, clusters=1024, seed=0)
    x, q = base.data, queries.data
    print(f"data {time.time() - t0:.1f}s", flush=True)
    t1 = time.time()
    graph = VamanaBuilder(degree_bound=32, build_worklist=64, sigma=1.2, seed=0).fit(x).graph_
    build_s = time.time() - t1
    print(f"VamanaBuilder {build_s:.1f}s", flush=True)
    t1 = time.time()
    cb = ProductQuantizer(m=32, iters=25, seed=0).fit(x).codebook_
    codes = compress_with_codebook(x, cb)
    print(f"PQ {time.time() - t1:.1f}s", flush=True)
    arrays = dict(
        base_sha256=np.array(sha(x)), queries=q.astype(np.float32), queries_sha256=np.array(sha(q)),
        n=np.int64(x.shape[0]), dim=np.int64(x.shape[1]), clusters=np.int64(1024), seed=np.int64(0),
        adjacency=graph.adjacency, degrees=graph.degrees, medoid=np.int64(graph.medoid),
        degree_bound=np.int64(graph.degree_bound),
        sub_sizes=np.asarray(cb.subspace_sizes, np.int32),
        centroids=np.concatenate([c.ravel() for c in cb.centroids]).astype(np.float32),
        codes=codes.codes, k=np.int64(10), bloom_entries=np.int64(399_887),
        t_values=np.asarray(T_VALUES, np.int64), build_seconds=np.float64(build_s),
        cores=np.int64(os.cpu_count() or 1))
    for t in T_VALUES:
        s = bang.GraphSearcher(k=10, t=t, mode="in_memory", bloom_entries=399_887,
                               batch_size=10_000, rerank=True, debug_checks=True)
        s.fit(x, graph=graph, codebook=cb, codes=codes)
        s.search(q[:50])  # warm (numba / numpy first-call costs)
        t1 = time.perf_counter()
        r = s.search(q)
        dt = time.perf_counter() - t1
        lens = np.array([len(v) for v in r.visit_logs], np.int64)
        offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        flat = np.concatenate([np.asarray(v, np.int32) for v in r.visit_logs])
        arrays.update({f"t{t}_ids": r.ids, f"t{t}_dists": r.dists, f"t{t}_iterations": r.iterations,
                       f"t{t}_short": r.short, f"t{t}_converged": r.converged,
                       f"t{t}_log_offsets": offs, f"t{t}_log_ids": flat,
                       f"t{t}_reference_qps": np.float64(q.shape[0] / dt)})
        print(f"t={t}: reference search {dt:.2f}s ({q.shape[0] / dt:.1f} QPS), "
              f"mean iters {r.iterations.mean():.1f}", flush=True)
    path = os.path.join(HERE, "c1_reference.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path}: {os.path.getsize(path) / 2**20:.1f} MiB in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
