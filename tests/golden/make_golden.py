"""Generate golden fixtures by running the READ-ONLY Python reference.

Run here (never on the GPU box -- /root/reference does not exist there):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports ``bang`` from /root/reference/pkg/src and writes small ``.npz``
fixtures next to this file.  Every fixture stores the reference's inputs and
the reference's own outputs, so tests can pin (1) the CPU oracle and (2) the
CUDA path against the reference without the reference being present.

Cases (reference call sites in /root/reference/pkg/src/bang/):
  search_*.npz  GraphSearcher(...).search   engine.py:409-452 (+ debug_checks)
  pq_table.npz  build_pq_dist_table         pq.py:299-319
  adc.npz       _pq_point_dists             engine.py:99-105
  bloom.npz     BloomFilterBank.filter_and_set / bit_positions  bloom.py:37-163
  kernels.npz   merge_sort_rows / merge_rows kernels.py:68-109
  exact.npz     exact_sq_dists / rerank     engine.py:48-51, 273-292
"""

from __future__ import annotations

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
from bang import engine as ref_engine  # noqa: E402
from bang.bloom import BloomFilterBank, bit_positions  # noqa: E402
from bang.datasets import gaussian_mixture  # noqa: E402
from bang.graph import GraphIndex, build_index, compute_medoid  # noqa: E402
from bang.kernels import SENTINEL, merge_rows, merge_sort_rows, pack_keys  # noqa: E402
from bang.pq import (PQCodebook, build_pq_dist_table, compress_with_codebook,  # noqa: E402
                     train_codebook)


def _save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}: {os.path.getsize(path) / 1024:.1f} KiB")


def _flatten_logs(logs):
    lens = np.array([len(x) for x in logs], np.int64)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    flat = np.concatenate([np.asarray(x, np.int64) for x in logs]) if len(logs) else np.zeros(0, np.int64)
    return offs, flat


def _search_case(name, base, queries, graph, codebook, codes, *, k, t, bloom, rerank=True,
                 modes=("in_memory",), batch_size=10_000, note=""):
    outs = {}
    for mode in modes:
        s = bang.GraphSearcher(k=k, t=t, mode=mode, bloom_entries=bloom,
                               batch_size=batch_size, rerank=rerank, debug_checks=True)
        if mode == "exact_distance":
            s.fit(base, graph=graph)
        else:
            s.fit(base, graph=graph, codebook=codebook, codes=codes)
        t0 = time.perf_counter()
        outs[mode] = s.search(queries)
        print(f"  {name} {mode}: {time.perf_counter() - t0:.2f}s")
    r = outs[modes[0]]
    for mode in modes[1:]:
        if mode == "exact_distance":
            continue
        o = outs[mode]
        assert np.array_equal(o.ids, r.ids) and np.array_equal(o.dists, r.dists)
        assert np.array_equal(o.iterations, r.iterations)
    offs, flat = _flatten_logs(r.visit_logs)
    arrays = dict(
        base=np.asarray(getattr(base, "data", base)),
        queries=np.asarray(getattr(queries, "data", queries), np.float32),
        adjacency=graph.adjacency, degrees=graph.degrees,
        medoid=np.int64(graph.medoid), degree_bound=np.int64(graph.degree_bound),
        k=np.int64(k), t=np.int64(t), bloom_entries=np.int64(bloom),
        rerank=np.bool_(rerank), mode=np.array(modes[0]),
        ids=r.ids, dists=r.dists, iterations=r.iterations, converged=r.converged,
        short=r.short, log_offsets=offs, log_ids=flat, note=np.array(note))
    if codebook is not None:
        arrays["sub_sizes"] = np.asarray(codebook.subspace_sizes, np.int32)
        arrays["centroids"] = np.concatenate([c.ravel() for c in codebook.centroids]).astype(np.float32)
        arrays["codes"] = codes.codes
    if "exact_distance" in outs:
        e = outs["exact_distance"]
        eo, ef = _flatten_logs(e.visit_logs)
        arrays.update(ex_ids=e.ids, ex_dists=e.dists, ex_iterations=e.iterations,
                      ex_short=e.short, ex_log_offsets=eo, ex_log_ids=ef)
    _save(name, **arrays)


def toy_fixture():
    # the 12-node worked example of tests/conftest.py:14-74 (paper Fig. 2)
    sys.path.insert(0, "/root/reference/pkg")
    import importlib.util
    spec = importlib.util.spec_from_file_location("ref_conftest", "/root/reference/pkg/tests/conftest.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    coords = np.zeros((12, 2), np.float32)
    for node, (xy, _, _) in mod.TOY_LAYOUT.items():
        coords[node] = xy
    cents = np.full((256, 2), 10_000.0, np.float32)
    for node, (xy, cluster, _) in mod.TOY_LAYOUT.items():
        cents[cluster] = xy
    cents[11] = (114.0, 86.0)
    cb = PQCodebook(dim=2, subspace_sizes=[2], centroids=[cents])
    codes = compress_with_codebook(coords, cb)
    graph = GraphIndex.from_lists([mod.TOY_ADJACENCY[i] for i in range(12)],
                                  medoid=mod.TOY_MEDOID, degree_bound=3)
    q = mod.TOY_QUERY[None, :]
    _search_case("search_toy_k2.npz", coords, q, graph, cb, codes, k=2, t=8, bloom=4096,
                 modes=("in_memory", "pipelined", "exact_distance"),
                 note="conftest.py toy; TOY_VISIT_ORDER")
    _search_case("search_toy_k8.npz", coords, q, graph, cb, codes, k=8, t=8, bloom=4096,
                 modes=("in_memory",), note="TOY_RERANKED")
    _search_case("search_toy_norerank.npz", coords, q, graph, cb, codes, k=2, t=8, bloom=4096,
                 rerank=False, modes=("in_memory",))


def random_graph(n, R, rng, min_deg=0):
    lists = []
    for i in range(n):
        deg = int(rng.integers(min_deg, R + 1))
        picks = rng.choice(n - 1, size=deg, replace=False)
        picks[picks >= i] += 1
        lists.append(picks.astype(np.int32))
    return lists


def search_fixtures():
    # (a) Vamana graph, f32, uniform subspaces (sub=4): the engine tests' shape
    base, queries = gaussian_mixture(3000, 48, 16, clusters=24, seed=101)
    graph = build_index(base.data, degree_bound=16, build_worklist=32, seed=101)
    cb = train_codebook(base, m=4, iters=8, seed=101)
    codes = compress_with_codebook(base.data, cb)
    _search_case("search_vamana_f32.npz", base.data, queries.data, graph, cb, codes,
                 k=10, t=24, bloom=399_887, modes=("in_memory", "pipelined", "exact_distance"))
    # same index, tiny Bloom filter: false positives + in-row slot collisions (replay path)
    _search_case("search_vamana_bloom61.npz", base.data, queries.data, graph, cb, codes,
                 k=5, t=16, bloom=61, modes=("in_memory",))
    _search_case("search_vamana_norerank.npz", base.data, queries.data, graph, cb, codes,
                 k=10, t=24, bloom=50_021, rerank=False, modes=("in_memory",))

    # (b) R = 64 (two neighbours per lane on the GPU), uneven subspaces 20 -> [3]*4+[2]*6? (m=8)
    base, queries = gaussian_mixture(2500, 40, 20, clusters=20, seed=202)
    graph = build_index(base.data, degree_bound=40, build_worklist=48, seed=202)
    cb = train_codebook(base, m=8, iters=6, seed=202)
    codes = compress_with_codebook(base.data, cb)
    _search_case("search_vamana_r40_uneven.npz", base.data, queries.data, graph, cb, codes,
                 k=10, t=40, bloom=399_887, modes=("in_memory",))

    # (c) uint8 vectors (SIFT-shape recipe of SURVEY.md 8(d)), m=8 (sub=4)
    b, q = gaussian_mixture(2000, 32, 32, clusters=20, seed=303)
    bu8 = np.clip(np.rint(32 * b.data + 128), 0, 255).astype(np.uint8)
    qf = np.clip(np.rint(32 * q.data + 128), 0, 255).astype(np.float32)
    graph = build_index(bu8, degree_bound=24, build_worklist=32, seed=303)
    cb = train_codebook(bu8, m=8, iters=6, seed=303)
    codes = compress_with_codebook(bu8, cb)
    _search_case("search_vamana_u8.npz", bu8, qf, graph, cb, codes, k=10, t=32,
                 bloom=399_887, modes=("in_memory",))

    # (d) random graph with degrees 0..64 (incl. degree-0 nodes), m=2 (sub=3), d=6;
    # a dense regime where worklists fill and truncation matters
    rng = np.random.default_rng(404)
    n, R = 1500, 64
    lists = random_graph(n, R, rng)
    base = rng.normal(size=(n, 6)).astype(np.float32)
    med = compute_medoid(base)
    if len(lists[med]) == 0:
        lists[med] = np.array([(med + 1) % n], np.int32)
    graph = GraphIndex.from_lists(lists, medoid=med, degree_bound=R)
    cb = train_codebook(base, m=2, iters=6, seed=404)
    codes = compress_with_codebook(base, cb)
    queries = rng.normal(size=(40, 6)).astype(np.float32)
    _search_case("search_random_r64.npz", base, queries, graph, cb, codes, k=7, t=20,
                 bloom=997, modes=("in_memory",))

    # (e) dead-end medoid: medoid of degree 0 converges after one expansion.
    # k=1: with k > next_pow2(max visit count) the reference itself raises
    # IndexError at engine.py:268 (its re-rank key matrix is narrower than k);
    # the B200 path pads with -1/+inf and sets short instead.
    lists2 = [np.asarray(x, np.int32) for x in lists]
    lists2[med] = np.zeros(0, np.int32)
    graph2 = GraphIndex.from_lists(lists2, medoid=med, degree_bound=R)
    _search_case("search_deadend.npz", base, queries[:4], graph2, cb, codes, k=1, t=8,
                 bloom=997, modes=("in_memory",))


def function_fixtures():
    rng = np.random.default_rng(7)
    # pq table: uneven sizes (9 dims, m=3 -> [3,3,3]) and (10 dims, m=4 -> [3,3,2,2])
    arrays = {}
    for tag, dim, m in (("a", 9, 3), ("b", 10, 4), ("c", 128, 32), ("d", 96, 48)):
        base = rng.normal(size=(600, dim)).astype(np.float32)
        cb = train_codebook(base, m=m, iters=3, seed=1)
        q = (rng.normal(size=(37, dim)) * 1.7).astype(np.float32)
        tab = build_pq_dist_table(q, cb).table
        arrays[f"{tag}_q"] = q
        arrays[f"{tag}_sizes"] = np.asarray(cb.subspace_sizes, np.int32)
        arrays[f"{tag}_centroids"] = np.concatenate([c.ravel() for c in cb.centroids])
        arrays[f"{tag}_table"] = tab
    _save("pq_table.npz", **arrays)

    # adc over random pairs
    table = rng.random((5, 16, 256)).astype(np.float32) * 100
    codes = rng.integers(0, 256, size=(300, 16), dtype=np.uint8)
    qrows = rng.integers(0, 5, size=2000)
    ids = rng.integers(0, 300, size=2000)
    d = ref_engine._pq_point_dists(table, qrows, codes[ids])
    _save("adc.npz", table=table, codes=codes, qrows=qrows, ids=ids, dists=d,
          keys=pack_keys(d, ids))

    # bloom: slots for pinned ids + bank sequences with collisions
    pin_ids = np.array([0, 1, 2, 10, 12345, 2**31 - 1, 999_999_999], np.int64)
    p1, p2 = bit_positions(pin_ids, 399_887)
    cases = {}
    for ci, (count, entries, nprobe, idmax) in enumerate(
            ((3, 17, 25, 100), (5, 997, 40, 5000), (4, 399_887, 200, 2**31 - 1),
             (2, 61, 64, 200), (1, 4096, 2, 5))):
        bank = BloomFilterBank(count, entries)
        rows_all, ids_all, fresh_all, splits = [], [], [], [0]
        for rep in range(6):
            rows = np.sort(rng.integers(0, count, size=nprobe))
            ids = rng.integers(0, idmax, size=nprobe)
            if ci == 4:
                rows, ids = np.zeros(2, np.int64), np.array([4, 4])
            fr = bank.filter_and_set(rows, ids)
            rows_all.append(rows); ids_all.append(ids); fresh_all.append(fr)
            splits.append(splits[-1] + rows.size)
        cases[f"c{ci}_count"] = np.int64(count)
        cases[f"c{ci}_entries"] = np.int64(entries)
        cases[f"c{ci}_rows"] = np.concatenate(rows_all)
        cases[f"c{ci}_ids"] = np.concatenate(ids_all).astype(np.int64)
        cases[f"c{ci}_fresh"] = np.concatenate(fresh_all)
        cases[f"c{ci}_splits"] = np.asarray(splits, np.int64)
        cases[f"c{ci}_bits"] = bank.bits.copy()
    _save("bloom.npz", pin_ids=pin_ids, pin_p1=p1, pin_p2=p2, **cases)

    # sort / merge rows (ties, sentinels, payload)
    n, w = 64, 32
    dd = rng.choice(np.float32([0.5, 1.0, 2.0, 3.5, 7.25]), size=(n, w))
    ii = rng.integers(0, 1_000_000, size=(n, w))
    keys = pack_keys(dd, ii)
    keys[rng.random((n, w)) < 0.2] = SENTINEL
    srt = merge_sort_rows(keys)
    a = merge_sort_rows(keys[:, :16].copy())
    b = merge_sort_rows(keys[:, 16:].copy())
    pay = rng.random((n, 16)) < 0.5
    mk, mp = merge_rows(a, b, a_payload=pay)
    _save("kernels.npz", keys=keys, sorted=srt, a=a, b=b, a_payload=pay,
          merged=mk, merged_payload=mp)

    # exact distances + rerank (f32 and u8)
    x = rng.normal(size=(500, 96)).astype(np.float32)
    q = rng.normal(size=(500, 96)).astype(np.float32)
    xu = rng.integers(0, 256, size=(500, 128)).astype(np.uint8)
    qu = rng.integers(0, 256, size=(500, 128)).astype(np.float32)
    ex = ref_engine.exact_sq_dists(x, q)
    exu = ref_engine.exact_sq_dists(xu, qu)
    cand = rng.choice(500, size=40, replace=False)
    rr_ids, rr_d, rr_short = ref_engine.rerank(cand, x[cand], q[0], k=10)
    _save("exact.npz", x=x, q=q, ex=ex, xu=xu, qu=qu, exu=exu, cand=cand,
          rr_ids=rr_ids, rr_dists=rr_d, rr_short=np.bool_(rr_short))


if __name__ == "__main__":
    t0 = time.time()
    function_fixtures()
    toy_fixture()
    search_fixtures()
    print(f"done in {time.time() - t0:.1f}s")
