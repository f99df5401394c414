"""GPU proximity-graph construction for the benchmark indexes (offline).

The reference builds with a sequential two-pass Vamana (graph.py:251-395),
~290 s at 100K points and days at 10M.  This builder keeps its
pruning rule -- RobustPrune with slack sigma (graph.py:118-147): keep the
closest live candidate v, drop every u with sigma^2 d(v,u) <= d(p,u) -- but
takes candidates from an exact k-NN pass and then adds pruned reverse edges,
all batched on the GPU with torch.  Output is the reference's GraphIndex
layout (padded (n, R) int32, -1 pads, degrees, medoid).  It is index
construction, not the hot path.
"""

from __future__ import annotations

import os

import numpy as np

from .._dev import torch_device
from ..graph import GraphIndex, compute_medoid


def knn(x, K: int, qchunk: int = 1024, bchunk: int = 1 << 21):
    """Exact K nearest neighbours of every row (self excluded): ids, sq dists."""
    import torch
    n = x.shape[0]
    K = min(K, n - 1)
    sq = x.square().sum(1)
    out_i = torch.empty((n, K), dtype=torch.int64, device=x.device)
    out_d = torch.empty((n, K), dtype=torch.float32, device=x.device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        for lo in range(0, n, qchunk):
            q = x[lo:lo + qchunk]
            rows = torch.arange(lo, lo + q.shape[0], device=x.device)
            best_d = best_i = None
            for blo in range(0, n, bchunk):
                d = sq[lo:lo + q.shape[0], None] + sq[None, blo:blo + bchunk] - 2.0 * (q @ x[blo:blo + bchunk].T)
                cols = torch.arange(blo, blo + d.shape[1], device=x.device)
                d[rows[:, None] == cols[None, :]] = float("inf")
                dv, di = torch.topk(d, min(K, d.shape[1]), dim=1, largest=False)
                di = di + blo
                if best_d is None:
                    best_d, best_i = dv, di
                else:
                    cd, ci = torch.cat([best_d, dv], 1), torch.cat([best_i, di], 1)
                    best_d, sel = torch.topk(cd, K, dim=1, largest=False)
                    best_i = torch.gather(ci, 1, sel)
            out_i[lo:lo + q.shape[0]] = best_i
            out_d[lo:lo + q.shape[0]] = best_d.clamp_min(0)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return out_i, out_d


def robust_prune(x, cand, dcand, R: int, sigma: float, chunk: int = 0):
    """Batched RobustPrune (graph.py:118-147) over candidate rows sorted by
    (distance, id); cand -1 = empty.  Returns (n, R) ids (-1 padded), degrees.
    The per-rank loop is sync-free (masked scatter), so a chunk costs a fixed
    number of launches whatever its contents."""
    import torch
    n, C = cand.shape
    sig2 = float(sigma) ** 2
    if not chunk:
        chunk = max(1024, min(32768, (1 << 31) // max(1, C * C * 4)))
    out = torch.full((n, R), -1, dtype=torch.int64, device=x.device)
    deg = torch.zeros(n, dtype=torch.int64, device=x.device)
    for lo in range(0, n, chunk):
        c = cand[lo:lo + chunk].long()
        dp = dcand[lo:lo + chunk]
        B = c.shape[0]
        alive = c >= 0
        v = x[c.clamp_min(0)].float()  # (B, C, d)
        vsq = v.square().sum(-1)
        D = vsq[:, :, None] + vsq[:, None, :] - 2.0 * torch.bmm(v, v.transpose(1, 2))
        del v
        kept = torch.full((B, R), -1, dtype=torch.int64, device=x.device)
        nk = torch.zeros(B, dtype=torch.int64, device=x.device)
        last = int((alive.sum(0) > 0).nonzero().max().item()) + 1 if bool(alive.any()) else 0
        for r in range(last):
            take = alive[:, r] & (nk < R)
            slot = nk.clamp_max(R - 1)[:, None]
            cur = kept.gather(1, slot).squeeze(1)
            kept.scatter_(1, slot, torch.where(take, c[:, r], cur)[:, None])
            nk += take.long()
            alive &= ~(take[:, None] & (sig2 * D[:, r, :] <= dp))
            alive[:, r] = False
        out[lo:lo + B] = kept
        deg[lo:lo + B] = nk
    return out, deg


def _sort_rows_by_dist(ids, d):
    import torch
    # ascending (dist, id): sort by id then stable by distance
    o1 = torch.argsort(ids, dim=1)
    ids, d = torch.gather(ids, 1, o1), torch.gather(d, 1, o1)
    o2 = torch.argsort(d, dim=1, stable=True)
    return torch.gather(ids, 1, o2), torch.gather(d, 1, o2)


def _pair_sqdist(x, a, b, chunk: int = 1 << 23):
    """|x[a] - x[b]|^2 for index vectors a, b, in bounded chunks."""
    import torch
    out = torch.empty(a.shape[0], dtype=torch.float32, device=x.device)
    for lo in range(0, a.shape[0], chunk):
        out[lo:lo + chunk] = (x[a[lo:lo + chunk]].float() - x[b[lo:lo + chunk]].float()).square().sum(1)
    return out


def add_reverse_edges(x, adj, deg, R: int, sigma: float, rev_cap: int | None = None):
    """For every edge p->q offer p to q; rows that overflow R are re-pruned."""
    import torch
    n = adj.shape[0]
    rev_cap = rev_cap or R
    valid = adj >= 0
    src = torch.arange(n, device=x.device)[:, None].expand_as(adj)[valid]
    dst = adj[valid]
    dd = _pair_sqdist(x, src, dst)
    # group by destination, nearest sources first; one stable sort on the
    # (dst, f32 bits of dd) key == stable sort by dd, then stable by dst
    key = (dst << 32) | dd.view(torch.int32).long()
    order = torch.sort(key, stable=True).indices
    del key
    src, dst, dd = src[order], dst[order], dd[order]
    del order
    counts = torch.bincount(dst, minlength=n)
    starts = torch.cumsum(counts, 0) - counts
    rank = torch.arange(dst.numel(), device=x.device) - starts[dst]
    keep = rank < rev_cap
    rev = torch.full((n, rev_cap), -1, dtype=torch.int64, device=x.device)
    revd = torch.full((n, rev_cap), float("inf"), device=x.device)
    rev[dst[keep], rank[keep]] = src[keep]
    revd[dst[keep], rank[keep]] = dd[keep]
    del src, dst, dd, rank, keep
    own_d = torch.full(adj.shape, float("inf"), dtype=torch.float32, device=x.device)
    rows = torch.arange(n, device=x.device)[:, None].expand_as(adj)
    own_d[valid] = _pair_sqdist(x, rows[valid], adj[valid])
    cand = torch.cat([adj, rev], 1)
    cd = torch.cat([own_d, revd], 1)
    del rev, revd, own_d
    # drop duplicates (mutual edges): keep one copy per id
    cs, o = torch.sort(cand, dim=1)
    dup = torch.zeros_like(cs, dtype=torch.bool)
    dup[:, 1:] = (cs[:, 1:] == cs[:, :-1]) & (cs[:, 1:] >= 0)
    dup = torch.zeros_like(dup).scatter_(1, o, dup)
    del cs, o
    cand = torch.where(dup, torch.full_like(cand, -1), cand)
    cd = torch.where(dup | (cand < 0), torch.full_like(cd, float("inf")), cd)
    cand = torch.where(torch.isinf(cd), torch.full_like(cand, -1), cand)
    cand, cd = _sort_rows_by_dist(cand, cd)
    cand = torch.where(torch.isinf(cd), torch.full_like(cand, -1), cand)
    total = (cand >= 0).sum(1)
    over = total > R
    new_adj = cand[:, :R].clone()
    new_deg = torch.minimum(total, torch.tensor(R, device=x.device))
    if bool(over.any()):
        idx = torch.nonzero(over).squeeze(1)
        pa, pd = robust_prune(x, cand[idx], cd[idx], R, sigma)
        new_adj[idx] = pa
        new_deg[idx] = pd
    return new_adj, new_deg


def _nearest_centroids(x, cent, k: int, chunk: int = 1 << 18):
    """ids (n, k) of the k nearest rows of cent for every row of x (f32)."""
    import torch
    csq = cent.square().sum(1)
    out = torch.empty((x.shape[0], k), dtype=torch.int64, device=x.device)
    for lo in range(0, x.shape[0], chunk):
        xb = x[lo:lo + chunk].float()
        d = csq[None, :] - 2.0 * (xb @ cent.T)
        out[lo:lo + chunk] = torch.topk(d, k, dim=1, largest=False).indices
    return out


def kmeans(x, nlist: int, iters: int = 10, sample: int = 1 << 20, seed: int = 0):
    """Lloyd k-means on a seeded sample (partitioning for the IVF k-NN)."""
    import torch
    n = x.shape[0]
    g = torch.Generator().manual_seed(seed)
    idx = torch.randperm(n, generator=g)[:min(n, max(sample, nlist))].to(x.device)
    xs = x[idx].float()
    cent = xs[torch.randperm(xs.shape[0], generator=g)[:nlist].to(x.device)].clone()
    for _ in range(iters):
        a = _nearest_centroids(xs, cent, 1)[:, 0]
        sums = torch.zeros_like(cent).index_add_(0, a, xs)
        cnt = torch.bincount(a, minlength=nlist).float()
        cent = torch.where(cnt[:, None] > 0, sums / cnt.clamp_min(1)[:, None], cent)
    return cent


def knn_ivf(x, K: int, nlist: int = 0, nprobe: int = 8, max_rows: int = 4096, seed: int = 0):
    """Approximate K-NN of every row (self excluded) in O(n * nprobe * n/nlist):
    k-means partitions; the rows of partition c are compared exactly (f32)
    against every row of the nprobe partitions whose centroids are nearest
    to c's.  Returns ids (n, K) int64 (-1 where fewer candidates) and squared
    distances (inf there).  Sub-quadratic replacement of knn() for the 10M+
    configs; graph construction only, not the hot path."""
    import torch
    n = x.shape[0]
    K = min(K, n - 1)
    nlist = nlist or max(1, min(n // 64, int(round(n / 1000))))
    nprobe = min(nprobe, nlist)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        cent = kmeans(x, nlist, seed=seed)
        assign = _nearest_centroids(x, cent, 1)[:, 0]
        probes = _nearest_centroids(cent, cent, nprobe).cpu().numpy()
        order = torch.argsort(assign, stable=True)
        counts = torch.bincount(assign, minlength=nlist).cpu().numpy()
        offs = np.concatenate([[0], np.cumsum(counts)])
        sq = x.float().square().sum(1)
        out_i = torch.full((n, K), -1, dtype=torch.int64, device=x.device)
        out_d = torch.full((n, K), float("inf"), dtype=torch.float32, device=x.device)
        for c in range(nlist):
            if counts[c] == 0:
                continue
            cand = torch.cat([order[offs[p]:offs[p + 1]] for p in probes[c] if counts[p]])
            xc = x[cand].float()
            kk = min(K, cand.shape[0] - 1)
            if kk < 1:
                continue
            for lo in range(offs[c], offs[c + 1], max_rows):
                mem = order[lo:min(offs[c + 1], lo + max_rows)]
                d = sq[mem][:, None] + sq[cand][None, :] - 2.0 * (x[mem].float() @ xc.T)
                d = torch.where(mem[:, None] == cand[None, :], float("inf"), d)
                dv, di = torch.topk(d, kk, dim=1, largest=False)
                out_i[mem, :kk] = torch.where(torch.isinf(dv), torch.full_like(di, -1), cand[di])
                out_d[mem, :kk] = dv.clamp_min(0)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return out_i, out_d


def locality_order(base, nlist: int = 0, seed: int = 0, device=None) -> np.ndarray:
    """Index layout: a node order in which graph neighbours sit close in
    memory.  k-means cells (about 1,000 points each) are chained greedily by
    nearest centroid, and nodes are laid out cell by cell, so the code rows,
    adjacency rows and vectors a search gathers for one region of space share
    L2 lines and DRAM pages.  Returns perm: new position -> old id.  Applying
    it (relabel_index) renames nodes only; the graph and the search over it
    are unchanged."""
    import torch
    dev = device if device is not None else torch_device()
    xn = np.asarray(base)
    n = xn.shape[0]
    nlist = nlist or max(1, n // 1000)
    x = torch.from_numpy(np.ascontiguousarray(xn)).to(dev)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        cent = kmeans(x, nlist, seed=seed)
        assign = torch.empty(n, dtype=torch.int64, device=dev)
        for lo in range(0, n, 1 << 21):
            assign[lo:lo + (1 << 21)] = _nearest_centroids(x[lo:lo + (1 << 21)].float(), cent, 1)[:, 0]
        # greedy nearest-neighbour chain through the centroids
        csq = cent.square().sum(1)
        d = csq[:, None] + csq[None, :] - 2.0 * (cent @ cent.T)
        used = torch.zeros(nlist, dtype=torch.bool, device=dev)
        rank = torch.empty(nlist, dtype=torch.int64, device=dev)
        cur = int(torch.argmin(csq))
        for r in range(nlist):
            rank[cur] = r
            used[cur] = True
            if r + 1 < nlist:
                cur = int(torch.argmin(torch.where(used, float("inf"), d[cur])))
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    key = rank[assign] * n + torch.arange(n, device=dev)
    return torch.argsort(key).cpu().numpy()


def relabel_index(perm: np.ndarray, base, adjacency, degrees, medoid: int, device=None):
    """Nodes renamed by perm (new position -> old id): returns (base, adjacency,
    degrees, medoid) in the new order; adjacency entries are renamed, -1
    padding kept."""
    import torch
    dev = device if device is not None else torch_device()
    n = perm.shape[0]
    p = torch.from_numpy(perm).to(dev)
    inv = torch.empty(n, dtype=torch.int32, device=dev)
    inv[p] = torch.arange(n, dtype=torch.int32, device=dev)
    adj = torch.from_numpy(np.ascontiguousarray(adjacency)).to(dev)[p]
    adj = torch.where(adj >= 0, inv[adj.clamp_min(0).long()], adj)
    deg = np.ascontiguousarray(np.asarray(degrees)[perm])
    out_base = np.ascontiguousarray(np.asarray(base)[perm])
    return out_base, adj.cpu().numpy(), deg, int(inv[int(medoid)])


def medoid_of(x, chunk: int = 1 << 21) -> int:
    """compute_medoid (graph.py:107-115) on the device: f64 mean, f64 distances."""
    import torch
    n = x.shape[0]
    mean = torch.zeros(x.shape[1], dtype=torch.float64, device=x.device)
    for lo in range(0, n, chunk):
        mean += x[lo:lo + chunk].double().sum(0)
    mean /= n
    best_v, best_i = None, 0
    for lo in range(0, n, chunk):
        d = (x[lo:lo + chunk].double() - mean).square().sum(1)
        v, i = torch.min(d, 0)
        if best_v is None or float(v) < best_v:
            best_v, best_i = float(v), lo + int(i)
    return best_i


def build_graph(base, degree_bound: int = 64, build_worklist: int = 200, sigma: float = 1.2,
                seed: int = 0, candidates: int | None = None, exact_limit: int = 2_000_000,
                device=None, log=None) -> GraphIndex:
    """k-NN candidates (2R by default) -> RobustPrune(sigma) -> reverse edges.
    Exact k-NN up to exact_limit points, partitioned (IVF) k-NN above."""
    import time
    import torch
    dev = device if device is not None else torch_device()
    xn = np.asarray(base)
    n = xn.shape[0]
    R = int(degree_bound)
    if n < 2:
        raise ValueError("need at least 2 points to build a graph")
    x = torch.from_numpy(np.ascontiguousarray(xn, dtype=np.float32)).to(dev)
    K = min(n - 1, candidates or max(2 * R, min(build_worklist, 3 * R)))
    t0 = time.time()
    if n <= exact_limit:
        ids, d = knn(x, K)
        medoid = compute_medoid(xn)
    else:
        ids, d = knn_ivf(x, K, seed=seed)
        medoid = medoid_of(x)
    t1 = time.time()
    # row sort in bounded chunks (the full-table argsorts and gathers would
    # need ~5x the (n, K) int64 table at once)
    for lo in range(0, n, 1 << 20):
        si, sd = _sort_rows_by_dist(ids[lo:lo + (1 << 20)], d[lo:lo + (1 << 20)])
        ids[lo:lo + (1 << 20)] = torch.where(torch.isinf(sd), torch.full_like(si, -1), si)
        d[lo:lo + (1 << 20)] = sd
        del si, sd
    adj, deg = robust_prune(x, ids, d, R, sigma)
    del ids, d
    t2 = time.time()
    adj, deg = add_reverse_edges(x, adj, deg, R, sigma)
    t3 = time.time()
    if log:
        log(f"[graph_build] n={n} knn {t1 - t0:.1f}s prune {t2 - t1:.1f}s reverse {t3 - t2:.1f}s")
    # the medoid must not be a dead end on a pathological input
    adj_np = adj.to(torch.int32).cpu().numpy()
    deg_np = deg.to(torch.int32).cpu().numpy()
    cols = np.arange(R)[None, :]
    adj_np[cols >= deg_np[:, None]] = -1
    return GraphIndex(adj_np, deg_np, medoid, R, validate=False)


def refine_graph(x, adj, deg, visit_fn, R: int, sigma: float = 1.2, chunk: int = 1 << 20,
                 max_cand: int = 192, log=None):
    """One batch-synchronous Vamana pass (graph.py:251-344 semantics, all
    points at once against the previous graph): for every point p the nodes
    its greedy search expands (visit_fn(lo, hi) -> CSR offsets/ids of the
    searches for points lo..hi-1) plus its current neighbours are the
    candidates; RobustPrune(sigma) keeps R; reverse edges are added and
    overflowing rows re-pruned.  adj/deg are torch tensors on x's device."""
    import time
    import torch
    n = x.shape[0]
    new_adj = torch.full((n, R), -1, dtype=torch.int64, device=x.device)
    new_deg = torch.zeros(n, dtype=torch.int64, device=x.device)
    t_search = t_prune = 0.0
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        t0 = time.time()
        offs, flat = visit_fn(lo, hi)
        t1 = time.time()
        b = hi - lo
        offs = torch.as_tensor(np.asarray(offs, np.int64), device=x.device)
        flat = torch.as_tensor(np.asarray(flat, np.int64), device=x.device)
        lens = offs[1:] - offs[:-1]
        W = int(lens.max().item()) if b else 0
        vis = torch.full((b, max(W, 1)), -1, dtype=torch.int64, device=x.device)
        rows = torch.repeat_interleave(torch.arange(b, device=x.device), lens)
        cols = torch.arange(flat.numel(), device=x.device) - offs[:-1][rows]
        vis[rows, cols] = flat
        cand = torch.cat([vis, adj[lo:hi].long()], 1)
        self_ids = torch.arange(lo, hi, device=x.device)[:, None]
        cand = torch.where(cand == self_ids, torch.full_like(cand, -1), cand)
        # unique per row
        cs, _ = torch.sort(cand, dim=1)
        dup = torch.zeros_like(cs, dtype=torch.bool)
        dup[:, 1:] = cs[:, 1:] == cs[:, :-1]
        cand = torch.where(dup, torch.full_like(cs, -1), cs)
        valid = cand >= 0
        cd = torch.full(cand.shape, float("inf"), dtype=torch.float32, device=x.device)
        rr = torch.arange(lo, hi, device=x.device)[:, None].expand_as(cand)
        cd[valid] = _pair_sqdist(x, rr[valid], cand[valid])
        cand, cd = _sort_rows_by_dist(cand, cd)
        cand, cd = cand[:, :max_cand], cd[:, :max_cand]
        cand = torch.where(torch.isinf(cd), torch.full_like(cand, -1), cand)
        a, d = robust_prune(x, cand, cd, R, sigma)
        new_adj[lo:hi] = a
        new_deg[lo:hi] = d
        t_search += t1 - t0
        t_prune += time.time() - t1
    t2 = time.time()
    new_adj, new_deg = add_reverse_edges(x, new_adj, new_deg, R, sigma)
    if log:
        log(f"[graph_build] refine: search {t_search:.1f}s prune {t_prune:.1f}s reverse {time.time() - t2:.1f}s")
    return new_adj, new_deg


def build_graph_partitioned(base, degree_bound: int = 64, parts: int = 16, overlap: int = 2,
                            sigma: float = 1.2, refine_fn=None, refine=(), seed: int = 0,
                            merge_chunk: int = 1 << 19, device=None, log=print, ckpt_dir=None) -> GraphIndex:
    """Graph of a base set too large for one build in HBM (C4: 100M x 128 u8).

    DiskANN-style partitioned construction: k-means on a sample gives
    `parts` centroids; every point joins its `overlap` nearest partitions;
    each partition gets its own graph (build_graph, then the search-based
    Vamana passes `refine_fn(members, local_graph, t)` for t in `refine`);
    a point's neighbour lists from its partitions are merged with one
    RobustPrune(sigma) over their union (exact distances).  Shared points
    connect the partitions.  Memory: the base stays in host RAM (u8 or f32)
    plus one partition and an (n, overlap*R) int32 candidate table.
    ckpt_dir: the assignment, the candidate table (a memory-mapped .npy)
    and the finished partitions are kept there; a later call resumes."""
    import gc
    import time
    import torch
    dev = device if device is not None else torch_device()
    xn = np.asarray(base)
    n, d = xn.shape
    R = int(degree_bound)
    t0 = time.time()
    ck = (lambda k: os.path.join(ckpt_dir, k)) if ckpt_dir else None
    if ckpt_dir:
        os.makedirs(ckpt_dir, exist_ok=True)
    if ck and os.path.exists(ck("assign.npy")):
        assign = np.load(ck("assign.npy"))
    else:
        rng = np.random.default_rng(seed)
        samp = np.sort(rng.choice(n, size=min(n, 1 << 20), replace=False))
        xs = torch.from_numpy(np.ascontiguousarray(xn[samp], dtype=np.float32)).to(dev)
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        try:
            cent = kmeans(xs, parts, seed=seed)
            del xs
            assign = np.empty((n, overlap), np.int32)
            for lo in range(0, n, 1 << 22):
                xb = torch.from_numpy(np.ascontiguousarray(xn[lo:lo + (1 << 22)])).to(dev).float()
                assign[lo:lo + (1 << 22)] = _nearest_centroids(xb, cent, overlap).to(torch.int32).cpu().numpy()
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev
        if ck:
            np.save(ck("assign.tmp.npy"), assign)
            os.replace(ck("assign.tmp.npy"), ck("assign.npy"))
    log(f"[graph_build] partitioned: {parts} parts x {overlap}-way, assignment {time.time() - t0:.1f}s")
    # members of each partition (stable order), and which of a point's slots it fills
    flat = assign.ravel()
    order = np.argsort(flat, kind="stable")
    bounds = np.searchsorted(flat[order], np.arange(parts + 1))
    done = set()
    if ck:
        if os.path.exists(ck("cand.npy")):
            cand = np.load(ck("cand.npy"), mmap_mode="r+")
            if os.path.exists(ck("done.txt")):
                done = {int(v) for v in open(ck("done.txt")).read().split()}
        else:
            cand = np.lib.format.open_memmap(ck("cand.npy"), mode="w+", dtype=np.int32, shape=(n, overlap * R))
            cand[:] = -1
        log(f"[graph_build] checkpoint {ckpt_dir}: partitions done {sorted(done)}")
    else:
        cand = np.full((n, overlap * R), -1, np.int32)
    for p in range(parts):
        if p in done:
            continue
        t1 = time.time()
        sel = order[bounds[p]:bounds[p + 1]]
        members, slot = sel // overlap, sel % overlap
        if members.size < 2:
            continue
        g = build_graph(xn[members], degree_bound=R, sigma=sigma, seed=seed, device=dev)
        for t in refine:
            g = refine_fn(members, g, t)
        adj = g.adjacency
        glob = np.where(adj >= 0, members[np.clip(adj, 0, None)], -1).astype(np.int32)
        for j in range(overlap):
            m_ = slot == j
            cand[members[m_], j * R:(j + 1) * R] = glob[m_]
        del g, adj, glob
        if ck:
            cand.flush()
            with open(ck("done.txt"), "a") as f:
                f.write(f"{p}\n")
        # the partition's device tensors must be gone before the next one
        # (a reference cycle would otherwise keep ~10 GB per partition alive)
        gc.collect()
        if torch.cuda.is_available():
            torch.cuda.empty_cache()
        mem = torch.cuda.memory_allocated() / 2**30 if torch.cuda.is_available() else 0.0
        log(f"[graph_build] partition {p + 1}/{parts}: {members.size} points, {time.time() - t1:.1f}s "
            f"(device memory in use {mem:.1f} GiB)")
    # merge: RobustPrune over the union of each point's partition lists
    t2 = time.time()
    x = torch.from_numpy(np.ascontiguousarray(xn)).to(dev)  # native dtype (u8: n*d bytes)
    adj_out = np.full((n, R), -1, np.int32)
    deg_out = np.zeros(n, np.int32)
    for lo in range(0, n, merge_chunk):
        hi = min(n, lo + merge_chunk)
        c = torch.from_numpy(cand[lo:hi]).to(dev).long()
        cs, _ = torch.sort(c, dim=1)
        dup = torch.zeros_like(cs, dtype=torch.bool)
        dup[:, 1:] = cs[:, 1:] == cs[:, :-1]
        c = torch.where(dup, torch.full_like(cs, -1), cs)
        rows = torch.arange(lo, hi, device=dev)[:, None].expand_as(c)
        valid = c >= 0
        dd = torch.full(c.shape, float("inf"), dtype=torch.float32, device=dev)
        dd[valid] = _pair_sqdist(x, rows[valid], c[valid])
        c, dd = _sort_rows_by_dist(c, dd)
        c = torch.where(torch.isinf(dd), torch.full_like(c, -1), c)
        a, dg = robust_prune(x, c, dd, R, sigma)
        adj_out[lo:hi] = a.to(torch.int32).cpu().numpy()
        deg_out[lo:hi] = dg.to(torch.int32).cpu().numpy()
    medoid = medoid_of(x)
    del x
    torch.cuda.empty_cache()
    adj_out[np.arange(R)[None, :] >= deg_out[:, None]] = -1
    log(f"[graph_build] partitioned merge {time.time() - t2:.1f}s, total {time.time() - t0:.1f}s "
        f"(mean degree {deg_out.mean():.1f})")
    return GraphIndex(adj_out, deg_out, medoid, R, validate=False)
