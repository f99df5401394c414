"""Exact k-NN ground truth on the GPU (the reference's brute_force_knn,
metrics.py:16-77): f32 inner-product candidates, exact f64 re-check of the
top k + pad, ascending (distance, id)."""

from __future__ import annotations

import numpy as np

from .._dev import torch_device


def brute_force_knn(base, queries, k: int, pad: int = 16, qchunk: int = 1024, bchunk: int = 1 << 21):
    import torch
    dev = torch_device()
    xb = torch.from_numpy(np.ascontiguousarray(base, dtype=np.float32)).to(dev)
    xq = torch.from_numpy(np.ascontiguousarray(queries, dtype=np.float32)).to(dev)
    nb, nq = xb.shape[0], xq.shape[0]
    kk = min(nb, k + pad)
    bsq = xb.square().sum(1)
    ids_out = np.empty((nq, k), np.int32)
    d_out = np.empty((nq, k), np.float32)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        for lo in range(0, nq, qchunk):
            q = xq[lo:lo + qchunk]
            best_d = best_i = None
            for blo in range(0, nb, bchunk):
                d = bsq[None, blo:blo + bchunk] - 2.0 * (q @ xb[blo:blo + bchunk].T)
                dv, di = torch.topk(d, min(kk, d.shape[1]), dim=1, largest=False)
                di = di + blo
                if best_d is None:
                    best_d, best_i = dv, di
                else:
                    cd = torch.cat([best_d, dv], 1)
                    ci = torch.cat([best_i, di], 1)
                    best_d, sel = torch.topk(cd, kk, dim=1, largest=False)
                    best_i = torch.gather(ci, 1, sel)
            cand = best_i
            diff = xb[cand].double() - q[:, None, :].double()
            ex = diff.square().sum(-1)
            # ascending (dist, id): sort by id, then stable by distance
            o1 = torch.argsort(cand, dim=1)
            ex1, c1 = torch.gather(ex, 1, o1), torch.gather(cand, 1, o1)
            o2 = torch.argsort(ex1, dim=1, stable=True)
            ids_out[lo:lo + q.shape[0]] = torch.gather(c1, 1, o2)[:, :k].cpu().numpy()
            d_out[lo:lo + q.shape[0]] = torch.gather(ex1, 1, o2)[:, :k].float().cpu().numpy()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return ids_out, d_out


def recall_at_k(result_ids: np.ndarray, gt_ids: np.ndarray, k: int) -> float:
    """metrics.py:80-95: mean |top-k(result) & top-k(gt)| / k."""
    r = np.asarray(result_ids)[:, :k]
    g = np.asarray(gt_ids)[:, :k]
    hits = sum(len(set(a.tolist()) & set(b.tolist())) for a, b in zip(r, g))
    return hits / (k * r.shape[0])
