"""GPU product-quantizer training and encoding (offline artifacts).

Same container contract as the reference's ProductQuantizer (pq.py:185-281):
m subspaces split by subspace_split, 256 centroids each, codes = index of
the nearest centroid (lowest index on ties).  Lloyd iterations run batched
over all subspaces with torch on the GPU; the artifacts are inputs to the
search and are shared verbatim with the reference arm of the benchmark.
"""

from __future__ import annotations

import numpy as np

from .._dev import torch_device
from ..pq import CENTROIDS_PER_SUBSPACE, CompressedVectors, PQCodebook, subspace_split


def _subspace_views(x, sizes):
    import torch
    width = max(sizes)
    m = len(sizes)
    out = torch.zeros((m, x.shape[0], width), dtype=torch.float32, device=x.device)
    pos = 0
    for s, sz in enumerate(sizes):
        out[s, :, :sz] = x[:, pos:pos + sz]
        pos += sz
    return out  # zero-padded to a common width: padding adds 0 to every distance


def train_codebook(base, m: int, iters: int = 25, seed: int = 0, sample: int = 262_144,
                   device=None) -> PQCodebook:
    import torch
    dev = device if device is not None else torch_device()
    x = np.asarray(base)
    n, dim = x.shape
    sizes = subspace_split(dim, m)
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(n, size=min(n, sample), replace=False))
    xs = torch.from_numpy(np.ascontiguousarray(x[idx], dtype=np.float32)).to(dev)
    sub = _subspace_views(xs, sizes)  # (m, ns, w)
    ns = sub.shape[1]
    k = CENTROIDS_PER_SUBSPACE
    if ns >= m * k:
        init = torch.from_numpy(rng.choice(ns, size=(m, k), replace=False)).to(dev)
    else:  # small training sets: k distinct rows per subspace, drawn independently
        init = torch.from_numpy(np.stack([rng.choice(ns, size=k, replace=ns < k) for _ in range(m)])).to(dev)
    cents = torch.gather(sub, 1, init[:, :, None].expand(m, k, sub.shape[2])).clone()
    for _ in range(iters):
        d = (sub.square().sum(-1, keepdim=True) - 2 * torch.bmm(sub, cents.transpose(1, 2))
             + cents.square().sum(-1)[:, None, :])
        assign = d.argmin(-1)  # (m, ns)
        sums = torch.zeros_like(cents).scatter_add_(1, assign[:, :, None].expand_as(sub), sub)
        cnt = torch.zeros((m, k), device=dev).scatter_add_(1, assign, torch.ones_like(assign, dtype=torch.float32))
        empty = cnt == 0
        cents = torch.where(empty[:, :, None], cents, sums / cnt.clamp_min(1)[:, :, None])
    cents = cents.cpu().numpy()
    return PQCodebook(dim=dim, subspace_sizes=sizes,
                      centroids=[np.ascontiguousarray(cents[s, :, :sz]) for s, sz in enumerate(sizes)])


def encode(base, codebook: PQCodebook, chunk: int = 262_144, device=None) -> CompressedVectors:
    """Nearest centroid per subspace, exact f64 distances (lowest id on ties)."""
    import torch
    dev = device if device is not None else torch_device()
    x = np.asarray(base)
    out = np.empty((x.shape[0], codebook.m), np.uint8)
    cents = [torch.from_numpy(c.astype(np.float64)).to(dev) for c in codebook.centroids]
    offs = codebook.offsets()
    for lo in range(0, x.shape[0], chunk):
        xb = torch.from_numpy(np.ascontiguousarray(x[lo:lo + chunk], dtype=np.float32)).to(dev).double()
        for s, (c, off, sz) in enumerate(zip(cents, offs, codebook.subspace_sizes)):
            d = ((xb[:, None, off:off + sz] - c[None, :, :]) ** 2).sum(-1)
            out[lo:lo + chunk, s] = d.argmin(1).to(torch.uint8).cpu().numpy()
    return CompressedVectors(out)
