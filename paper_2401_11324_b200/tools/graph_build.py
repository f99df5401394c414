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


def robust_prune(x, cand, dcand, R: int, sigma: float, chunk: int = 8192):
    """Batched RobustPrune (graph.py:118-147) over candidate rows sorted by
    (distance, id); cand -1 = empty.  Returns (n, R) ids (-1 padded), degrees."""
    import torch
    n, C = cand.shape
    sig2 = float(sigma) ** 2
    out = torch.full((n, R), -1, dtype=torch.int64, device=x.device)
    deg = torch.zeros(n, dtype=torch.int64, device=x.device)
    for lo in range(0, n, chunk):
        c = cand[lo:lo + chunk]
        dp = dcand[lo:lo + chunk]
        B = c.shape[0]
        alive = c >= 0
        v = x[c.clamp_min(0)]  # (B, C, d)
        vsq = v.square().sum(-1)
        D = vsq[:, :, None] + vsq[:, None, :] - 2.0 * torch.bmm(v, v.transpose(1, 2))
        kept = torch.full((B, R), -1, dtype=torch.int64, device=x.device)
        nk = torch.zeros(B, dtype=torch.int64, device=x.device)
        ar = torch.arange(B, device=x.device)
        for r in range(C):
            take = alive[:, r] & (nk < R)
            if not bool(take.any()):
                if not bool(alive[:, r + 1:].any()):
                    break
                continue
            kept[ar[take], nk[take]] = c[take, r]
            nk += take.long()
            kill = take[:, None] & (sig2 * D[:, r, :] <= dp)
            alive &= ~kill
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


def add_reverse_edges(x, adj, deg, R: int, sigma: float, rev_cap: int | None = None):
    """For every edge p->q offer p to q; rows that overflow R are re-pruned."""
    import torch
    n = adj.shape[0]
    rev_cap = rev_cap or R
    valid = adj >= 0
    src = torch.arange(n, device=x.device)[:, None].expand_as(adj)[valid]
    dst = adj[valid]
    dd = (x[src] - x[dst]).square().sum(1)
    # group by destination, nearest sources first
    order = torch.argsort(dd, stable=True)
    src, dst, dd = src[order], dst[order], dd[order]
    order = torch.argsort(dst, stable=True)
    src, dst, dd = src[order], dst[order], dd[order]
    counts = torch.bincount(dst, minlength=n)
    starts = torch.cumsum(counts, 0) - counts
    rank = torch.arange(dst.numel(), device=x.device) - starts[dst]
    keep = rank < rev_cap
    rev = torch.full((n, rev_cap), -1, dtype=torch.int64, device=x.device)
    revd = torch.full((n, rev_cap), float("inf"), device=x.device)
    rev[dst[keep], rank[keep]] = src[keep]
    revd[dst[keep], rank[keep]] = dd[keep]
    own_d = torch.where(valid, (x[adj.clamp_min(0)] - x[:, None, :]).square().sum(-1),
                        torch.full_like(adj, float("inf"), dtype=torch.float32))
    cand = torch.cat([adj, rev], 1)
    cd = torch.cat([own_d, revd], 1)
    # drop duplicates (mutual edges): keep one copy per id
    cs, o = torch.sort(cand, dim=1)
    dup = torch.zeros_like(cs, dtype=torch.bool)
    dup[:, 1:] = (cs[:, 1:] == cs[:, :-1]) & (cs[:, 1:] >= 0)
    dup = torch.zeros_like(dup).scatter_(1, o, dup)
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


def build_graph(base, degree_bound: int = 64, build_worklist: int = 200, sigma: float = 1.2,
                seed: int = 0, candidates: int | None = None) -> GraphIndex:
    """k-NN candidates (2R by default) -> RobustPrune(sigma) -> reverse edges."""
    import torch
    dev = torch_device()
    xn = np.asarray(base)
    n = xn.shape[0]
    R = int(degree_bound)
    if n < 2:
        raise ValueError("need at least 2 points to build a graph")
    x = torch.from_numpy(np.ascontiguousarray(xn, dtype=np.float32)).to(dev)
    K = min(n - 1, candidates or max(2 * R, min(build_worklist, 3 * R)))
    ids, d = knn(x, K)
    ids, d = _sort_rows_by_dist(ids, d)
    adj, deg = robust_prune(x, ids, d, R, sigma)
    adj, deg = add_reverse_edges(x, adj, deg, R, sigma)
    medoid = compute_medoid(xn)
    # the medoid must not be a dead end on a pathological input
    adj_np = adj.cpu().numpy().astype(np.int32)
    deg_np = deg.cpu().numpy().astype(np.int32)
    cols = np.arange(R)[None, :]
    adj_np[cols >= deg_np[:, None]] = -1
    return GraphIndex(adj_np, deg_np, medoid, R, validate=False)
