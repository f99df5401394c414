"""GPU parity: every kernel of libbang.so against the reference's golden
outputs and the pinned CPU oracle (oracle/bang_oracle.c).

Bar (north_star): integer/index results bit-exact (visit logs, iterations,
top-k ids, short flags, Bloom bits); f32 distances exact here as well (the
arithmetic order is restated), with the stated tolerance 1e-4 relative only
used where noted.
"""

import os

import numpy as np
import pytest

import golden_util as gu
from oracle import oracle as O

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2401_11324_b200")


def _searcher_from_golden(g, mode="in_memory", **kw):
    cents = gu.split_centroids(g["centroids"], g["sub_sizes"])
    cb = B.PQCodebook(dim=g["base"].shape[1], subspace_sizes=[int(s) for s in g["sub_sizes"]],
                      centroids=cents)
    graph = B.GraphIndex(g["adjacency"], g["degrees"], int(g["medoid"]), int(g["degree_bound"]))
    params = dict(k=int(g["k"]), t=int(g["t"]), mode=mode, bloom_entries=int(g["bloom_entries"]),
                  rerank=bool(g["rerank"]), debug_checks=True)
    params.update(kw)
    s = B.GraphSearcher(**params)
    if mode == "exact_distance":
        s.fit(g["base"], graph=graph)
    else:
        s.fit(g["base"], graph=graph, codebook=cb, codes=B.CompressedVectors(g["codes"]))
    return s


def _assert_same(res, ids, dists, iters, logs, short=None):
    assert np.array_equal(res.iterations, iters)
    assert len(res.visit_logs) == len(logs)
    for a, b in zip(res.visit_logs, logs):
        assert np.array_equal(a, b)
    assert np.array_equal(res.ids, ids)
    assert np.array_equal(res.dists, dists)
    if short is not None:
        assert np.array_equal(res.short, short)
    assert res.converged.all()


# ----------------------------------------------------------------- kernels

def test_kernel1_pq_table_exact():
    g = gu.load("pq_table.npz")
    for tag in "abcd":
        cents = gu.split_centroids(g[f"{tag}_centroids"], g[f"{tag}_sizes"])
        cb = B.PQCodebook(dim=g[f"{tag}_q"].shape[1], subspace_sizes=[int(s) for s in g[f"{tag}_sizes"]],
                          centroids=cents)
        got = B.build_pq_dist_table(g[f"{tag}_q"], cb).table
        assert np.array_equal(got, g[f"{tag}_table"]), tag


def test_kernel2_bloom_bank_matches_reference_sequences():
    g = gu.load("bloom.npz")
    for case in range(5):
        count, entries = int(g[f"c{case}_count"]), int(g[f"c{case}_entries"])
        bank = B.BloomFilterBank(count, entries)
        sp = g[f"c{case}_splits"]
        for a, b in zip(sp[:-1], sp[1:]):
            fr = bank.filter_and_set(g[f"c{case}_rows"][a:b], g[f"c{case}_ids"][a:b])
            assert np.array_equal(fr, g[f"c{case}_fresh"][a:b]), case
        assert np.array_equal(bank.bits, g[f"c{case}_bits"]), case


def test_kernel2_bloom_collision_stress_vs_oracle():
    # 17-slot filters force in-row slot sharing on nearly every batch
    rng = np.random.default_rng(3)
    for entries in (17, 61, 997):
        bank = B.BloomFilterBank(6, entries)
        bits = np.zeros((6, (entries + 63) // 64), np.uint64)
        for _ in range(20):
            rows = rng.integers(0, 6, size=150)
            ids = rng.integers(0, 300, size=150)
            got = bank.filter_and_set(rows, ids)
            want = O.bloom_filter_and_set(bits, entries, rows, ids)
            assert np.array_equal(got, want)
        assert np.array_equal(bank.bits, bits)


def test_kernel2_set_all_rows_and_duplicates():
    bank = B.BloomFilterBank(4, 512)
    bank.set_all_rows(9)
    assert bank.filter_and_set(np.arange(4), np.full(4, 9)).tolist() == [False] * 4
    bank = B.BloomFilterBank(1, 4096)
    assert bank.filter_and_set(np.zeros(2, np.int64), np.array([4, 4])).tolist() == [True, False]


def test_kernel3_adc_exact():
    g = gu.load("adc.npz")
    tab = B.PQDistTable(g["table"])
    for q in range(tab.rho):
        sel = g["qrows"] == q
        got = B.asymmetric_distances(B.CompressedVectors(g["codes"]), g["ids"][sel], q, tab)
        assert np.array_equal(got, g["dists"][sel])


def test_kernel3_adc_vectorised_code_rows():
    # m = 32 and m = 48 take the 16-byte code-row path
    rng = np.random.default_rng(5)
    for m in (32, 48, 7):
        table = (rng.random((3, m, 256)) * 50).astype(np.float32)
        codes = rng.integers(0, 256, size=(500, m), dtype=np.uint8)
        ids = rng.integers(0, 500, size=3000)
        rows = rng.integers(0, 3, size=3000)
        want = O.adc(table, codes, rows, ids)
        tab = B.PQDistTable(table)
        for q in range(3):
            got = B.asymmetric_distances(B.CompressedVectors(codes), ids[rows == q], q, tab)
            assert np.array_equal(got, want[rows == q])


@pytest.mark.parametrize("d,m", [(128, 32), (96, 48), (20, 8)])
def test_kernel3_adc_pairs_query_grouped(d, m):
    """bang_adc_pairs_device (table built in shared memory per query) equals
    the oracle's table + sequential ADC, including empty pair ranges (m = 48
    code rows are 64-byte padded on the device)."""
    import torch
    from paper_2401_11324_b200 import _lib
    from paper_2401_11324_b200.tools.pq_train import encode, train_codebook
    rng = np.random.default_rng(d + m)
    n = 16_000
    base = rng.normal(size=(n, d)).astype(np.float32)
    cb = train_codebook(base, m=m, iters=3, seed=1)
    codes = encode(base, cb).codes
    graph = B.GraphIndex(np.zeros((n, 4), np.int32), np.zeros(n, np.int32), 0, 4)
    s = B.GraphSearcher(k=1, t=4, mode="in_memory")
    s.fit(base, graph=graph, codebook=cb, codes=B.CompressedVectors(codes))
    assert _lib.lib().bang_index_code_stride(s.index_.handle) == (64 if m == 48 else m)
    nq = 37
    q = rng.normal(size=(nq, d)).astype(np.float32)
    counts = rng.integers(0, 700, size=nq)
    counts[[3, 17]] = 0
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    ids = rng.integers(0, n, size=int(off[-1])).astype(np.uint32)
    table = O.pq_table(q, cb.centroids, cb.subspace_sizes)
    rows = np.repeat(np.arange(nq), counts)
    want = O.pack_keys(O.adc(table, codes, rows, ids.astype(np.int64)), ids.astype(np.int64))
    dev = torch.device("cuda", 0)
    dq = torch.from_numpy(q).to(dev)
    doff = torch.from_numpy(off).to(dev)
    dids = torch.from_numpy(ids.view(np.int32)).to(dev)
    dk = torch.empty(int(off[-1]), dtype=torch.int64, device=dev)
    _lib.check(_lib.lib().bang_adc_pairs_device(s.index_.handle, _lib.ptr(dq), nq, _lib.ptr(doff), _lib.ptr(dids),
                                                _lib.ptr(dk), None))
    torch.cuda.synchronize()
    assert np.array_equal(dk.cpu().numpy().view(np.uint64), np.asarray(want, np.uint64))


def test_kernel1_pq_table_host_entry():
    """bang_pq_table (host buffers, the handle's codebook) equals the
    reference's build_pq_dist_table (pq.py:299-319)."""
    g = gu.load("pq_table.npz")
    for tag in "cd":
        q = g[f"{tag}_q"]
        cents = gu.split_centroids(g[f"{tag}_centroids"], g[f"{tag}_sizes"])
        cb = B.PQCodebook(dim=q.shape[1], subspace_sizes=[int(s) for s in g[f"{tag}_sizes"]], centroids=cents)
        n = 64
        codes = B.CompressedVectors(np.zeros((n, cb.m), np.uint8))
        graph = B.GraphIndex(np.zeros((n, 4), np.int32), np.zeros(n, np.int32), 0, 4)
        s = B.GraphSearcher(k=1, t=4, mode="in_memory").fit(np.zeros((n, q.shape[1]), np.float32), graph=graph,
                                                           codebook=cb, codes=codes)
        assert np.array_equal(s.index_.pq_table(q), g[f"{tag}_table"]), tag


def test_kernel4_sort_and_merge_rows():
    g = gu.load("kernels.npz")
    assert np.array_equal(B.merge_sort_rows(g["keys"]), g["sorted"])
    mk, mp = B.merge_rows(g["a"], g["b"], a_payload=g["a_payload"])
    assert np.array_equal(mk, g["merged"]) and np.array_equal(mp, g["merged_payload"])
    # the paper's Fig. 4 instance (test_kernels.py:59-66)
    a = [(10, 2.0), (11, 9.0), (12, 21.0), (28, 28.0)]
    b = [(20, 4.0), (21, 7.0), (22, 12.0), (23, 16.0)]
    assert B.parallel_merge(a, b).index((28, np.float32(28.0))) == 7


def test_kernel4_worklist_update_matches_engine_step():
    """engine.py:201-217 on random worklist states (test_state.py:52-77 style)."""
    from paper_2401_11324_b200 import _dev, _lib
    rng = np.random.default_rng(0)
    for t, w in ((8, 4), (24, 32), (40, 64), (100, 64), (200, 128)):
        rows = 64
        wl = np.full((rows, t), O.SENTINEL, np.uint64)
        vis = np.zeros((rows, t), np.uint8)
        new = np.full((rows, w), O.SENTINEL, np.uint64)
        for r in range(rows):
            n_wl = int(rng.integers(1, t + 1))
            n_new = int(rng.integers(0, w + 1))
            ids = rng.choice(100_000, size=n_wl + n_new, replace=False)
            d = rng.integers(0, 50, size=n_wl + n_new).astype(np.float32)
            keys = O.pack_keys(d, ids)
            wl[r, :n_wl] = np.sort(keys[:n_wl])
            vis[r, :n_wl] = rng.random(n_wl) < 0.6
            new[r, rng.permutation(w)[:n_new]] = keys[n_wl:]
        # oracle (engine.py:201-217)
        head = np.where(vis.astype(bool), O.SENTINEL, wl).min(1)
        win_ref = np.minimum(new.min(1), head)
        merged, mvis = O.merge_rows(wl, O.sort_rows(new), a_payload=vis)
        kept, kvis = merged[:, :t], mvis[:, :t]
        done_ref = np.all(kvis | (kept == O.SENTINEL), axis=1)
        dwl, dvis, dnew = _dev.to_dev(wl), _dev.to_dev(vis), _dev.to_dev(new)
        dwin, ddone = _dev.empty((rows,), np.uint64), _dev.empty((rows,), np.uint8)
        _lib.check(_lib.lib().bang_worklist_update_device(
            _lib.ptr(dwl), _lib.ptr(dvis), rows, t, _lib.ptr(dnew), w, _lib.ptr(dwin), _lib.ptr(ddone),
            _lib.stream_ptr(_dev.stream())))
        assert np.array_equal(_dev.to_host(dwl, np.uint64), kept), (t, w)
        assert np.array_equal(_dev.to_host(dvis).astype(bool), kvis), (t, w)
        assert np.array_equal(_dev.to_host(dwin, np.uint64), win_ref), (t, w)
        assert np.array_equal(_dev.to_host(ddone).astype(bool), done_ref), (t, w)


def test_kernel5_exact_dists_and_rerank():
    g = gu.load("exact.npz")
    assert np.array_equal(B.exact_sq_dists(g["x"], g["q"]), g["ex"])
    assert np.array_equal(B.exact_sq_dists(g["xu"], g["qu"]), g["exu"])
    ids, d, short = B.rerank(g["cand"], g["x"][g["cand"]], g["q"][0], k=10)
    assert ids.tolist() == g["rr_ids"].tolist()
    assert np.array_equal(d, g["rr_dists"]) and bool(short) == bool(g["rr_short"])


def test_kernel5_rerank_device_entry_csr():
    from paper_2401_11324_b200 import _dev, _lib
    rng = np.random.default_rng(9)
    n, d, nq, k = 2000, 24, 50, 7
    x = rng.normal(size=(n, d)).astype(np.float32)
    q = rng.normal(size=(nq, d)).astype(np.float32)
    lens = rng.integers(0, 40, size=nq)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cand = np.concatenate([rng.choice(n, size=int(L), replace=False) for L in lens]).astype(np.int32)
    dx, dq, doff, dc = _dev.to_dev(x), _dev.to_dev(q), _dev.to_dev(offs), _dev.to_dev(cand)
    oi, od, osh = _dev.empty((nq, k), np.int32), _dev.empty((nq, k), np.float32), _dev.empty((nq,), np.uint8)
    _lib.check(_lib.lib().bang_rerank_device(_lib.ptr(dx), 0, d, _lib.ptr(dq), nq, _lib.ptr(doff), _lib.ptr(dc),
                                             k, _lib.ptr(oi), _lib.ptr(od), _lib.ptr(osh),
                                             _lib.stream_ptr(_dev.stream())))
    gi, gd, gs = _dev.to_host(oi), _dev.to_host(od), _dev.to_host(osh)
    for i in range(nq):
        c = cand[offs[i]:offs[i + 1]].astype(np.int64)
        wi = np.full(k, -1, np.int32)
        wd = np.full(k, np.inf, np.float32)
        cnt = O.lib().bo_rerank(O._ptr(c), c.size, O._ptr(x), 0, d, O._ptr(q[i]), k, O._ptr(wi), O._ptr(wd))
        assert np.array_equal(gi[i], wi) and np.array_equal(gd[i], wd)
        assert bool(gs[i]) == (c.size < k)


# ------------------------------------------------------------------ search

@pytest.mark.parametrize("name", gu.search_cases())
def test_search_matches_reference_golden(name):
    g = gu.load(name)
    res = _searcher_from_golden(g).search(g["queries"])
    _assert_same(res, g["ids"], g["dists"], g["iterations"], gu.logs(g["log_offsets"], g["log_ids"]),
                 g["short"])


@pytest.mark.parametrize("name", ["search_toy_k2.npz", "search_vamana_f32.npz", "search_vamana_u8.npz"])
def test_pipelined_equals_in_memory_and_reference(name):
    """test_engine.py:88-104: host-resident graph gives identical outputs."""
    g = gu.load(name)
    res = _searcher_from_golden(g, mode="pipelined").search(g["queries"])
    _assert_same(res, g["ids"], g["dists"], g["iterations"], gu.logs(g["log_offsets"], g["log_ids"]))


@pytest.mark.parametrize("variant,code", [("hbm-table", 1), ("codebook", 0), ("smem-table", 3)])
@pytest.mark.parametrize("name", ["search_toy_k2.npz", "search_vamana_f32.npz", "search_vamana_r40_uneven.npz",
                                  "search_random_r64.npz", "search_vamana_bloom61.npz", "search_vamana_u8.npz"])
def test_every_adc_variant_matches(name, variant, code):
    """All ADC data flows (HBM table from kernel 1, shared codebook, per-query
    smem table) give the reference's results bit for bit."""
    g = gu.load(name)
    s = _searcher_from_golden(g).set_adc_variant(variant)
    res = s.search(g["queries"])
    assert s.last_stats()["adc_variant"] == code
    _assert_same(res, g["ids"], g["dists"], g["iterations"], gu.logs(g["log_offsets"], g["log_ids"]))


@pytest.mark.parametrize("name", ["search_toy_k2.npz", "search_vamana_f32.npz"])
def test_exact_distance_mode_matches_reference(name):
    g = gu.load(name)
    res = _searcher_from_golden(g, mode="exact_distance").search(g["queries"])
    _assert_same(res, g["ex_ids"], g["ex_dists"], g["ex_iterations"],
                 gu.logs(g["ex_log_offsets"], g["ex_log_ids"]), g["ex_short"])


def test_toy_trace_and_kneighbors():
    g = gu.load("search_toy_k2.npz")
    s = _searcher_from_golden(g)
    res = s.search(g["queries"])
    assert res.visit_logs[0].tolist() == [6, 8, 7, 2, 5, 9, 11, 10]
    assert set(res.ids[0].tolist()) == {10, 8}
    dists, ids = s.kneighbors(g["queries"], n_neighbors=2)
    assert set(ids[0].tolist()) == {10, 8}


def test_batch_split_and_repeat_invariance():
    """test_engine.py:107-134."""
    g = gu.load("search_vamana_f32.npz")
    r1 = _searcher_from_golden(g, batch_size=7).search(g["queries"])
    r2 = _searcher_from_golden(g, batch_size=10_000).search(g["queries"])
    r3 = _searcher_from_golden(g, batch_size=10_000).search(g["queries"])
    for r in (r1, r3):
        assert np.array_equal(r.ids, r2.ids) and np.array_equal(r.dists, r2.dists)
        assert np.array_equal(r.iterations, r2.iterations)


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_non_finite_queries_rejected_on_device(bad):
    """validation.py:17-19: f32 queries are checked by bang_search on the
    device (the host skips its pass); same exception and message, and the
    handle stays usable."""
    g = gu.load("search_vamana_f32.npz")
    s = _searcher_from_golden(g)
    q = np.array(g["queries"], np.float32, copy=True)
    q[len(q) // 2, -1] = bad
    with pytest.raises(B.ParameterError, match="queries contains non-finite values"):
        s.search(q)
    with pytest.raises(B.ParameterError, match="queries contains non-finite values"):
        s.search(q.astype(np.float64))  # host check before the f32 cast
    res = s.search(g["queries"])
    _assert_same(res, g["ids"], g["dists"], g["iterations"], gu.logs(g["log_offsets"], g["log_ids"]))


def test_engine_equals_rerank_of_visit_log():
    """test_engine.py:137-149."""
    g = gu.load("search_vamana_r40_uneven.npz")
    res = _searcher_from_golden(g).search(g["queries"])
    for i in range(len(res.visit_logs)):
        log = res.visit_logs[i]
        ids, dists, short = B.rerank(log, g["base"][log], g["queries"][i], k=int(g["k"]))
        assert res.ids[i].tolist() == ids.tolist()
        assert np.array_equal(res.dists[i], dists)


def test_empty_batch_and_param_errors():
    g = gu.load("search_toy_k2.npz")
    s = _searcher_from_golden(g)
    r = s.search(np.zeros((0, 2), np.float32))
    assert r.ids.shape == (0, 2) and r.elapsed == 0.0
    with pytest.raises(B.ParameterError):
        s.search(np.zeros((1, 5), np.float32))
    with pytest.raises(B.ParameterError):
        s.search(g["queries"], k=9)


def _random_case(seed, n, d, R, m, nq, dtype=np.float32):
    from paper_2401_11324_b200.tools.datasets import gaussian_mixture, to_u8
    from paper_2401_11324_b200.tools.graph_build import build_graph
    from paper_2401_11324_b200.tools.pq_train import encode, train_codebook
    base, q = gaussian_mixture(n, nq, d, clusters=max(8, n // 100), seed=seed)
    if dtype == np.uint8:
        base, q = to_u8(base), to_u8(q).astype(np.float32)
    graph = build_graph(base, degree_bound=R, seed=seed)
    cb = train_codebook(base, m=m, iters=6, seed=seed)
    return base, q, graph, cb, encode(base, cb)


# (ADC flags, kernel option) combinations: every data flow of every kernel
_VARIANTS = [("auto", "auto"), ("smem-table", "auto"), ("smem-table", "warp"), ("codebook", "auto"),
             ("hbm-table", "auto"), ("smem-table", "cta")]


def _oracle_search(q, graph, cb, codes, base, t, z=399_887, rerank=True, k=10):
    return O.search(q, centroids=cb.centroids, sub_sizes=cb.subspace_sizes, codes=codes.codes,
                    adjacency=graph.adjacency, degrees=graph.degrees, medoid=graph.medoid, vectors=base,
                    k=k, t=t, bloom_entries=z, rerank=rerank, threads=8)


def _same_as_oracle(res, want):
    _assert_same(res, want["ids"], want["dists"], want["iterations"], want["visit_logs"], want["short"])


@pytest.mark.parametrize("seed,n,d,R,m,t,dtype", [
    (1, 20_000, 128, 64, 32, 64, np.uint8),   # C2 shape at reduced n: sub=4, m=32 fast path
    (2, 20_000, 96, 64, 48, 48, np.float32),  # C3 shape at reduced n: sub=2, m=48 fast path
    (3, 8_000, 40, 100, 10, 150, np.float32),  # R > 64 (4 neighbours per lane), uneven, t=150
])
def test_search_matches_oracle_generated(seed, n, d, R, m, t, dtype):
    base, q, graph, cb, codes = _random_case(seed, n, d, R, m, 300, dtype)
    s = B.GraphSearcher(k=10, t=t, mode="in_memory", bloom_entries=399_887, debug_checks=True)
    s.fit(base, graph=graph, codebook=cb, codes=codes)
    want = _oracle_search(q, graph, cb, codes, base, t)
    vec = m in (32, 48)
    if vec:
        s.set_adc_variant("auto").set_kernel("auto").search(q[:4])
        assert s.last_stats()["kernel"] == 8  # row + list warps per query, smem table (HBM graph)
    for variant, kernel in _VARIANTS:
        if kernel == "cta" and not vec:
            continue
        res = s.set_adc_variant(variant).set_kernel(kernel).search(q)
        _same_as_oracle(res, want)
    if vec:
        res = s.set_adc_variant("auto").set_kernel("split").search(q)
        assert s.last_stats()["kernel"] == 8
        _same_as_oracle(res, want)


@pytest.mark.parametrize("seed,n,d,R,m,t,dtype,z", [
    (16, 16_000, 96, 64, 48, 64, np.float32, 251),
    (17, 16_000, 128, 64, 32, 48, np.uint8, 1021),
    (18, 16_000, 96, 64, 48, 40, np.float32, 4099),
])
@pytest.mark.parametrize("flow", ["cta", "cta-summary", "split", "split-noprefetch", "split-exact"])
def test_cta_kernel_bloom_replay_matches_oracle(seed, n, d, R, m, t, dtype, z, flow):
    """CTA kernels with small Bloom filters: most rows share slots, so the
    warp replay from pre-state bits (replay_row_warp) runs constantly.
    cta: search_cta_kernel (filter cleared per query; -summary: smem bitmap of
    written words instead); split: search_split_kernel (with and without the
    head-row L2 prefetch; -exact: every row through the pre-state read, no
    fetch-or-only rows)."""
    base, q, graph, cb, codes = _random_case(seed, n, d, R, m, 300, dtype)
    s = B.GraphSearcher(k=10, t=t, mode="in_memory", bloom_entries=z, debug_checks=True)
    s.fit(base, graph=graph, codebook=cb, codes=codes)
    if flow.startswith("cta"):
        s.set_kernel("cta", bloom_clear=0 if flow == "cta-summary" else 1)
    else:
        s.set_kernel("split", row_prefetch=0 if flow == "split-noprefetch" else 1,
                     bloom_direct=0 if flow == "split-exact" else 1)
    want = _oracle_search(q, graph, cb, codes, base, t, z)
    res = s.search(q)
    assert s.last_stats()["kernel"] == (2 if flow.startswith("cta") else 8)
    _same_as_oracle(res, want)


# ---- the benchmarked operating point's code paths (merge chunks
# c >= 1 of the split kernel's list warps at t > 64 and of search_cta_kernel
# at t > NT)
# on C3-shaped indexes of 100K nodes (10M x 96 f32 shape, R=64, m=48) and a
# C2-shaped one (128-d u8, m=32)

_BIG = {}


def _big_case(shape):
    if shape not in _BIG:
        if shape == "C3":
            _BIG[shape] = _random_case(21, 100_000, 96, 64, 48, 160, np.float32)
        else:
            _BIG[shape] = _random_case(22, 100_000, 128, 64, 32, 160, np.uint8)
    return _BIG[shape]


_ORACLE = {}


def _big_oracle(shape, t, z=399_887):
    key = (shape, t, z)
    if key not in _ORACLE:
        base, q, graph, cb, codes = _big_case(shape)
        _ORACLE[key] = _oracle_search(q, graph, cb, codes, base, t, z)
    return _ORACLE[key]


@pytest.mark.parametrize("shape,t", [("C3", 100), ("C3", 166), ("C3", 256), ("C2", 80), ("C2", 200)])
def test_split_kernel_large_t_matches_oracle(shape, t):
    """search_split_kernel at worklists spanning 2-4 merge chunks of its 64
    list threads (t=166 is the C3 benchmark's operating point)."""
    base, q, graph, cb, codes = _big_case(shape)
    s = B.GraphSearcher(k=10, t=t, mode="in_memory", bloom_entries=399_887, debug_checks=True)
    s.fit(base, graph=graph, codebook=cb, codes=codes)
    res = s.set_kernel("split").search(q)
    assert s.last_stats()["kernel"] == 8
    _same_as_oracle(res, _big_oracle(shape, t))


@pytest.mark.parametrize("z", [20_011, 399_887])
@pytest.mark.parametrize("direct,head_row", [(0, 1), (1, 1), (1, 0)])
def test_split_bloom_direct_rows_match_oracle(z, direct, head_row):
    """bloom_direct: rows without in-row slot sharing (a per-(index, z)
    bitset) take their pre-state bits from the fetch-or, the others the
    pre-state read + replay.  z = 20,011 flags about a third of the rows, so
    one query mixes both paths; every 5th row repeats a neighbour id (always
    shared).  A second z on the same index rebuilds the bitset."""
    base, q, graph, cb, codes = _random_case(31, 20_000, 96, 64, 48, 200, np.float32)
    adj = graph.adjacency.copy()
    rows = np.arange(0, adj.shape[0], 5)
    adj[rows, 7] = adj[rows, 3]
    graph = B.GraphIndex(adj, graph.degrees, graph.medoid, graph.degree_bound, validate=False)
    s = B.GraphSearcher(k=10, t=100, mode="in_memory", bloom_entries=z, debug_checks=True)
    s.fit(base, graph=graph, codebook=cb, codes=codes)
    s.set_kernel("split", bloom_direct=direct, head_row=head_row)
    for zz in (z, 4099, z):
        s.bloom_entries = zz
        res = s.search(q)
        assert s.last_stats()["kernel"] == 8
        _same_as_oracle(res, _oracle_search(q, graph, cb, codes, base, 100, zz))


def test_index_prepare_then_search():
    """bang_index_prepare builds the split kernel's row flags ahead of the
    search (fit does it for the searcher's Bloom size); results unchanged."""
    base, q, graph, cb, codes = _random_case(31, 20_000, 96, 64, 48, 100, np.float32)
    s = B.GraphSearcher(k=10, t=64, mode="in_memory", bloom_entries=20_011, debug_checks=True)
    s.fit(base, graph=graph, codebook=cb, codes=codes)
    L = B._lib.lib()
    B._lib.check(L.bang_index_prepare(s.index_.handle, 4099))
    with pytest.raises(B.ParameterError):
        B._lib.check(L.bang_index_prepare(s.index_.handle, 0))
    for z in (20_011, 4099):
        s.bloom_entries = z
        res = s.set_kernel("split").search(q)
        _same_as_oracle(res, _oracle_search(q, graph, cb, codes, base, 64, z))


@pytest.mark.parametrize("seed,n,d,R,m,t,dtype", [
    (23, 16_000, 96, 100, 48, 120, np.float32),  # 64 < R <= 128: two slots per row thread
    (24, 16_000, 128, 128, 32, 200, np.uint8),
    (25, 16_000, 96, 40, 48, 30, np.float32),    # R < 64: idle row threads
])
def test_wide_and_narrow_rows_match_oracle(seed, n, d, R, m, t, dtype):
    base, q, graph, cb, codes = _random_case(seed, n, d, R, m, 200, dtype)
    s = B.GraphSearcher(k=10, t=t, mode="in_memory", bloom_entries=399_887, debug_checks=True)
    s.fit(base, graph=graph, codebook=cb, codes=codes)
    want = _oracle_search(q, graph, cb, codes, base, t)
    for kernel, kid in (("split", 8), ("cta", 2)):
        res = s.set_kernel(kernel).search(q)
        assert s.last_stats()["kernel"] == kid
        _same_as_oracle(res, want)


@pytest.mark.parametrize("t,k", [(1, 1), (10, 10), (11, 10)])
@pytest.mark.parametrize("kernel", ["split", "cta"])
def test_cta_kernels_tiny_worklists_match_oracle(t, k, kernel):
    """t = k down to 1: the threshold is the single entry, heads run out at once."""
    base, q, graph, cb, codes = _random_case(26, 8_000, 96, 64, 48, 100, np.float32)
    s = B.GraphSearcher(k=k, t=t, mode="in_memory", bloom_entries=399_887, debug_checks=True)
    s.fit(base, graph=graph, codebook=cb, codes=codes)
    for rerank in (True, False):
        s.rerank = rerank
        res = s.set_kernel(kernel).search(q)
        _same_as_oracle(res, _oracle_search(q, graph, cb, codes, base, t, rerank=rerank, k=k))


@pytest.mark.parametrize("kernel", ["split", "cta"])
def test_cta_kernels_without_rerank_match_oracle(kernel):
    """rerank=False: the outputs are the final worklist's first k entries."""
    base, q, graph, cb, codes = _big_case("C3")
    s = B.GraphSearcher(k=10, t=120, mode="in_memory", bloom_entries=399_887, rerank=False, debug_checks=True)
    s.fit(base, graph=graph, codebook=cb, codes=codes)
    res = s.set_kernel(kernel).search(q)
    _same_as_oracle(res, _oracle_search(q, graph, cb, codes, base, 120, rerank=False))


@pytest.mark.parametrize("shape,t", [("C3", 160), ("C3", 300), ("C2", 160), ("C2", 300)])
def test_cta_kernel_large_t_matches_oracle(shape, t):
    """search_cta_kernel at worklists spanning 2-3 merge chunks of NT = 128."""
    base, q, graph, cb, codes = _big_case(shape)
    s = B.GraphSearcher(k=10, t=t, mode="in_memory", bloom_entries=399_887, debug_checks=True)
    s.fit(base, graph=graph, codebook=cb, codes=codes)
    res = s.set_kernel("cta").search(q)
    assert s.last_stats()["kernel"] == 2
    _same_as_oracle(res, _big_oracle(shape, t))


@pytest.mark.parametrize("seed,n,d,R,m,t,dtype", [
    (14, 16_000, 128, 64, 32, 48, np.uint8),
    (15, 16_000, 96, 64, 48, 64, np.float32),
])
def test_pipelined_cta_kernel_matches_oracle(seed, n, d, R, m, t, dtype):
    """Graph + vectors in pinned, mapped host memory (mode="pipelined"): the
    split kernel (rows with a [deg,0,0,0] header read over PCIe) and the CTA
    kernel, both with the staged re-rank: identical to the oracle."""
    base, q, graph, cb, codes = _random_case(seed, n, d, R, m, 300, dtype)
    s = B.GraphSearcher(k=10, t=t, mode="pipelined", bloom_entries=399_887, debug_checks=True)
    s.fit(base, graph=graph, codebook=cb, codes=codes)
    want = _oracle_search(q, graph, cb, codes, base, t)
    for kernel, kid in (("auto", 2), ("cta", 2), ("split", 8)):
        res = s.set_kernel(kernel).search(q)
        assert s.last_stats()["kernel"] == kid
        _same_as_oracle(res, want)


@pytest.mark.parametrize("kernel", ["cta", "split"])
def test_cta_kernels_overflow_retry_is_exact(kernel):
    from paper_2401_11324_b200 import _lib
    base, q, graph, cb, codes = _random_case(10, 16_000, 96, 64, 48, 200, np.float32)
    t = 64
    s = B.GraphSearcher(k=10, t=t, mode="in_memory", bloom_entries=399_887).set_kernel(kernel)
    s.fit(base, graph=graph, codebook=cb, codes=codes)
    _lib.check(_lib.lib().bang_index_set_log_capacity(s.index_.handle, 60))
    res = s.search(q)
    assert s.last_stats()["retries"] > 0
    _same_as_oracle(res, _oracle_search(q, graph, cb, codes, base, t))


def test_explicit_kernel_rejects_unsupported_shapes():
    g = gu.load("search_vamana_f32.npz")  # m=4: no 16-byte code rows
    s = _searcher_from_golden(g).set_kernel("cta")
    with pytest.raises(B.ParameterError):
        s.search(g["queries"])
    with pytest.raises(B.ParameterError):
        s.set_kernel("no-such-kernel")


def test_visit_log_overflow_retry_is_exact():
    """Queries that expand more nodes than the device log holds are re-run
    with a wider log; results stay identical (t large, tiny Bloom filter)."""
    from paper_2401_11324_b200 import _lib
    base, q, graph, cb, codes = _random_case(4, 6_000, 16, 32, 4, 40, np.float32)
    t = 64
    s = B.GraphSearcher(k=10, t=t, mode="in_memory", bloom_entries=399_887)
    s.fit(base, graph=graph, codebook=cb, codes=codes)
    _lib.check(_lib.lib().bang_index_set_log_capacity(s.index_.handle, 50))
    res = s.search(q)
    assert s.last_stats()["retries"] > 0
    want = O.search(q, centroids=cb.centroids, sub_sizes=cb.subspace_sizes, codes=codes.codes,
                    adjacency=graph.adjacency, degrees=graph.degrees, medoid=graph.medoid, vectors=base,
                    k=10, t=t, bloom_entries=399_887, threads=8)
    _assert_same(res, want["ids"], want["dists"], want["iterations"], want["visit_logs"], want["short"])


def test_stats_counters_are_consistent():
    g = gu.load("search_vamana_f32.npz")
    s = _searcher_from_golden(g)
    res = s.search(g["queries"])
    st = s.last_stats()
    assert st["iterations"] == int(res.iterations.sum())
    assert st["rerank_cands"] == int(res.iterations.sum())
    # probes = sum of expanded degrees
    deg = g["degrees"]
    assert st["probes"] == int(sum(deg[log].sum() for log in res.visit_logs))
    assert st["kernel_ms"] > 0



@pytest.mark.parametrize("cap", [2048, 40])
def test_public_search_readback_paths(cap):
    """GraphSearcher.search reads results back in one batch when its
    page-locked log buffer covers nq x the device log capacity; a larger
    capacity (cap=2048 > max(1024, 4t)) takes the two-call protocol, a small
    one (overflow re-runs) the general path.  All equal to the oracle."""
    from paper_2401_11324_b200 import _lib
    base, q, graph, cb, codes = _random_case(28, 8_000, 96, 64, 48, 150, np.float32)
    t = 48
    s = B.GraphSearcher(k=10, t=t, mode="in_memory", bloom_entries=399_887, debug_checks=True)
    s.fit(base, graph=graph, codebook=cb, codes=codes)
    want = _oracle_search(q, graph, cb, codes, base, t)
    res = s.search(q)  # default capacity: the one-batch path
    _same_as_oracle(res, want)
    _lib.check(_lib.lib().bang_index_set_log_capacity(s.index_.handle, cap))
    res = s.search(q)
    _same_as_oracle(res, want)
    assert (s.last_stats()["retries"] > 0) == (cap < 60)
