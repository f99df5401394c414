"""Kernel-3 micro-benchmark: bang_adc_pairs_device over synthetic
query-grouped pairs (random ids into a 10M-row code table, ~11.6K pairs per
query as in the C3 benchmark search), one line per kernel variant
(BANG_ADC_PAIRS env), outputs cross-checked between variants and against the
oracle on a few queries.

    python scripts/adc_micro.py [--n 10000000] [--m 48] [--dim 96] [--nq 10000]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--m", type=int, default=48)
    ap.add_argument("--dim", type=int, default=96)
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--pairs", type=int, default=11_600, help="mean pairs per query")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--variants", default="staged,lanes")
    ap.add_argument("--once", action="store_true", help="one launch per variant (for ncu)")
    a = ap.parse_args()

    import torch
    import paper_2401_11324_b200 as B
    from paper_2401_11324_b200 import _lib
    from oracle import oracle as O

    rng = np.random.default_rng(0)
    sub = a.dim // a.m
    cents = [rng.normal(size=(256, sub)).astype(np.float32) for _ in range(a.m)]
    cb = B.PQCodebook(dim=a.dim, subspace_sizes=[sub] * a.m, centroids=cents)
    codes = rng.integers(0, 256, size=(a.n, a.m), dtype=np.uint8)
    graph = B.GraphIndex(np.zeros((a.n, 1), np.int32), np.zeros(a.n, np.int32), 0, 1)
    base = np.zeros((a.n, a.dim), np.uint8)
    s = B.GraphSearcher(k=1, t=4, mode="in_memory")
    s.fit(base, graph=graph, codebook=cb, codes=B.CompressedVectors(codes))
    del base
    dev = torch.device("cuda", 0)
    q = rng.normal(size=(a.nq, a.dim)).astype(np.float32)
    counts = rng.integers(int(a.pairs * 0.8), int(a.pairs * 1.2) + 1, size=a.nq)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    P = int(off[-1])
    g = torch.Generator(device=dev).manual_seed(1)
    dids = torch.randint(0, a.n, (P,), device=dev, dtype=torch.int32, generator=g)
    dq = torch.from_numpy(q).to(dev)
    doff = torch.from_numpy(off).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(dev)
    L = _lib.lib()
    h = s.index_.handle

    # oracle on the first 3 queries
    nchk = 3
    ids_chk = dids[: int(off[nchk])].cpu().numpy().astype(np.int64)
    table = O.pq_table(q[:nchk], cb.centroids, cb.subspace_sizes)
    rows = np.repeat(np.arange(nchk), counts[:nchk])
    want = np.asarray(O.pack_keys(O.adc(table, codes, rows, ids_chk), ids_chk), np.uint64)

    results, ref_keys = [], None
    for var in a.variants.split(","):
        os.environ["BANG_ADC_PAIRS"] = var
        keys = torch.empty(P, dtype=torch.int64, device=dev)

        def launch():
            _lib.check(L.bang_adc_pairs_device(h, _lib.ptr(dq), a.nq, _lib.ptr(doff), _lib.ptr(dids),
                                               _lib.ptr(keys), _lib.stream_ptr(stream)), "adc_pairs")

        launch()
        torch.cuda.synchronize()
        got = keys[: int(off[nchk])].cpu().numpy().view(np.uint64)
        ok = bool(np.array_equal(got, want))
        if ref_keys is None:
            ref_keys = keys
            same = True
        else:
            same = bool(torch.equal(keys, ref_keys))
        ms = []
        for _ in range(0 if a.once else a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                launch()
                e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = float(np.mean(ms)) if ms else float("nan")
        algo = P * (a.m + 12) + a.nq * 4 * a.dim
        gbs = algo / (t / 1e3) / 1e9
        r = dict(variant=var, n=a.n, m=a.m, pairs=P, ms=round(t, 4), gpairs_s=round(P / t / 1e6, 2),
                 gbs=round(gbs, 1), frac=round(gbs / 6457.4, 4), oracle_ok=ok, same_as_first=same)
        print(json.dumps(r), flush=True)
        results.append(r)
        if var != a.variants.split(",")[0]:
            del keys
    if not all(r["oracle_ok"] and r["same_as_first"] for r in results):
        sys.exit(1)


if __name__ == "__main__":
    main()
