"""Benchmark of the B200 batched graph search (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference] [--config C3]

One "step" = one batched search of the config's query batch (10K queries; the
default config is C3, BASELINE.json's 10M-point target) at the smallest worklist size t whose recall@10 >= 0.9 (chosen by a
sweep before timing).  Reported:
  value  QPS with queries/outputs resident in HBM (bang_search_device), the
         sum of per-step CUDA-event times on the launching stream, L2 flushed
         (256 MiB memset) between steps outside the events, max over ranks;
  e2e    QPS through the public API GraphSearcher.search with the queries in
         pinned host memory (H2D, search, D2H of ids/dists/iterations/short/
         visit logs inside the timed region);
  roofline  the fused search kernel's algorithmic HBM bytes / its event time;
  cpu_baseline  the CPU oracle (oracle/, a C port of the reference path, all
         host threads) on the same queries (the parity run, timed).
  parity  the oracle's result for the whole batch at the operating point,
         compared bit for bit (ids, dists, iterations, short, visit logs);
         a mismatch fails the run (exit 3).
Multi-GPU (torchrun): --scaling weak (default): each rank searches its own
10K-query batch; --scaling strong: one 10K batch split over the ranks (the
reference's batch split, engine.py:431-443).  The index is replicated; no
collective on the search path.  --config C1 runs BASELINE configs[0] on the
reference's own artifacts (tests/golden/c1_reference.npz).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

T_SWEEP = (10, 12, 16, 20, 24, 32, 40, 48, 64, 80, 96, 112, 128, 144, 160, 176, 200, 224, 256)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if len(s) >= 6 and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 6 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples if len(s) >= 6 for i in range(4)
                          if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def recall(ids, gt, k=10):
    if gt is None:  # throughput-only configs (no ground truth)
        return None
    from paper_2401_11324_b200.tools.groundtruth import recall_at_k
    return recall_at_k(ids, gt, k)


def oracle_kwargs(art, t, k, bloom, threads):
    g = art["graph"]
    cb = art["codebook"]
    return dict(centroids=cb.centroids, sub_sizes=cb.subspace_sizes, codes=art["codes"].codes,
                adjacency=g.adjacency, degrees=g.degrees, medoid=g.medoid, vectors=art["base"], k=k, t=t,
                bloom_entries=bloom, threads=threads)


def cpu_oracle_run(art, queries, t, k, bloom, threads=None):
    """The CPU oracle (oracle/, a C port of the reference path, OpenMP over
    queries) over the given queries: (result, seconds, threads)."""
    from oracle import oracle as O
    O.build()
    threads = threads or os.cpu_count() or 1
    t0 = time.perf_counter()
    res = O.search(queries, **oracle_kwargs(art, t, k, bloom, threads))
    return res, time.perf_counter() - t0, threads


def parity_check(res, want, visit_logs=True):
    """Bit-exact comparison of a GPU SearchResult with the oracle's result
    (ids, dists, iterations, short, and every visit log as a sequence)."""
    nq = res.ids.shape[0]
    bad = np.zeros(nq, bool)
    bad |= ~np.all(res.ids == want["ids"], axis=1)
    bad |= ~np.all(res.dists.view(np.uint32) == want["dists"].view(np.uint32), axis=1)
    bad |= res.iterations != want["iterations"]
    bad |= res.short != want["short"]
    if visit_logs:
        for i in range(nq):
            if not bad[i] and not np.array_equal(res.visit_logs[i], want["visit_logs"][i]):
                bad[i] = True
    return {"queries": int(nq), "mismatches": int(bad.sum()),
            "first_mismatch": int(np.argmax(bad)) if bad.any() else None,
            "compared": "ids, dists (bits), iterations, short, visit logs (sequences)" if visit_logs
                        else "ids, dists (bits), iterations, short"}


def adc_pairs_roofline(searcher, art, queries, res, dev, stream, flush, peak, peak_kind, reps=3):
    """Times kernel 3 (adc_pairs_kernel) over the pairs of the benchmark
    search: for each query, the rows of every node it expanded (its Bloom
    probes), in visit order.  Achieved = pairs x (m + 12) B / kernel time."""
    import torch
    from paper_2401_11324_b200 import _lib
    g = art["graph"]
    offs, flat = res.visit_logs.csr()
    m = art["codebook"].m
    adj = torch.from_numpy(np.ascontiguousarray(g.adjacency)).to(dev)
    deg = torch.from_numpy(np.ascontiguousarray(g.degrees)).to(dev).long()
    v = torch.from_numpy(np.asarray(flat, np.int64)).to(dev)
    rows = adj[v]                                   # (visits, R)
    mask = torch.arange(g.adjacency.shape[1], device=dev)[None, :] < deg[v][:, None]
    ids = rows[mask].contiguous()                   # probes in visit order
    per_visit = mask.sum(1)
    qo = torch.from_numpy(np.asarray(offs, np.int64)).to(dev)
    csum = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), torch.cumsum(per_visit, 0)])
    pair_off = csum[qo].contiguous()
    del adj, rows, mask
    dq = torch.from_numpy(np.ascontiguousarray(queries, np.float32)).to(dev)
    keys = torch.empty(ids.numel(), dtype=torch.int64, device=dev)
    L = _lib.lib()
    h = searcher.index_.handle
    nq = dq.shape[0]

    def launch():
        _lib.check(L.bang_adc_pairs_device(h, _lib.ptr(dq), nq, _lib.ptr(pair_off), _lib.ptr(ids),
                                           _lib.ptr(keys), _lib.stream_ptr(stream)), "bang_adc_pairs_device")

    launch()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launch()
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = float(np.mean(ms))
    pairs = int(ids.numel())
    algo = pairs * (m + 12) + nq * (4 * queries.shape[1])
    ach = algo / (t / 1000.0) / 1e9
    return {"kernel": "bang::adc_pairs_kernel", "pairs": pairs, "queries": int(nq), "ms": round(t, 4),
            "bytes_per_pair": m + 12, "algorithmic_bytes": algo, "achieved": round(ach, 1), "peak": peak,
            "unit": "GB/s", "frac": round(ach / peak, 4), "peak_kind": peak_kind,
            "pairs_source": "every (query, neighbour) probe of the benchmark search, grouped by query "
                            "(the rows of each query's visit log); table built in smem per query",
            "l2": "flushed before each timed launch"}


def load_c1_reference(log):
    """BASELINE configs[0] with the reference's OWN artifacts
    (tests/golden/c1_reference.npz, written by tests/golden/make_c1.py with
    VamanaBuilder / ProductQuantizer / GraphSearcher); base regenerated from
    the seed (SHA-256 checked)."""
    import hashlib
    from paper_2401_11324_b200 import CompressedVectors, GraphIndex, PQCodebook
    from paper_2401_11324_b200.tools.datasets import gaussian_mixture
    from paper_2401_11324_b200.tools.groundtruth import brute_force_knn
    with np.load(os.path.join(ROOT, "tests", "golden", "c1_reference.npz")) as z:
        g = {k: z[k] for k in z.files}
    base, q = gaussian_mixture(int(g["n"]), g["queries"].shape[0], int(g["dim"]), clusters=int(g["clusters"]),
                               seed=int(g["seed"]))
    assert hashlib.sha256(base.tobytes()).hexdigest() == str(g["base_sha256"]), "C1 base vectors differ"
    sizes = [int(x) for x in g["sub_sizes"]]
    cents, pos = [], 0
    for sz in sizes:
        cents.append(g["centroids"][pos:pos + 256 * sz].reshape(256, sz))
        pos += 256 * sz
    gt_ids, gt_d = brute_force_knn(base, g["queries"], 10)
    log("[bench] C1: reference artifacts from tests/golden/c1_reference.npz")
    meta = dict(desc="synthetic 100Kx128 fp32 Gaussian mixture (clusters=1024), the reference's VamanaBuilder "
                     "R=32 L=64 graph and ProductQuantizer m=32 codebook, 1K queries, k=10",
                n=int(g["n"]), dim=int(g["dim"]), dtype="f32", R=int(g["degree_bound"]), m=len(sizes),
                clusters=1024, reference_outputs={int(t): g for t in g["t_values"]})
    return dict(base=base, queries=g["queries"], graph=GraphIndex(g["adjacency"], g["degrees"], int(g["medoid"]),
                                                                int(g["degree_bound"])),
                codebook=PQCodebook(dim=int(g["dim"]), subspace_sizes=sizes, centroids=cents),
                codes=CompressedVectors(g["codes"]), gt_ids=gt_ids, gt_dists=gt_d, meta=meta,
                ref=g)


def select_t(search_fn, queries, gt, target, k, t_fixed):
    """Smallest t in T_SWEEP whose recall@10 >= target, refined by bisection
    between the last two sweep points (unit granularity)."""
    sweep = []
    if t_fixed:
        return t_fixed, sweep
    t_sel = 0
    for t in T_SWEEP:
        ids, iters = search_fn(t)
        r = recall(ids, gt, k)
        sweep.append({"t": t, "recall": round(r, 4), "mean_iters": float(np.mean(iters))})
        if r >= target:
            t_sel = t
            break
    if not t_sel:
        return T_SWEEP[-1], sweep
    if len(sweep) > 1:
        lo, hi = sweep[-2]["t"], t_sel
        while hi - lo > 1:
            mid = (lo + hi) // 2
            ids, iters = search_fn(mid)
            r = recall(ids, gt, k)
            sweep.append({"t": mid, "recall": round(r, 4), "mean_iters": float(np.mean(iters))})
            if r >= target:
                hi = mid
            else:
                lo = mid
        t_sel = hi
    return t_sel, sweep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--config", default=os.environ.get("BANG_BENCH_CONFIG", "C3"))
    ap.add_argument("--scaling", default="weak", choices=("weak", "strong"),
                    help="weak: every rank searches its own query batch; strong: one batch split over the ranks")
    ap.add_argument("--t", type=int, default=0, help="fixed worklist size (default: recall sweep)")
    ap.add_argument("--target-recall", type=float, default=0.9)
    ap.add_argument("--bloom", type=int, default=399_887)
    ap.add_argument("--cache", default=os.environ.get("BANG_BENCH_CACHE", "/tmp/bang_bench_cache"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle comparison at the operating point")
    ap.add_argument("--profile", action="store_true", help="1 warm step + 1 step for ncu; no baselines")
    ap.add_argument("--phases", action="store_true", help="per-phase cycle profile (diagnostic)")
    ap.add_argument("--variant", default="auto", choices=("auto", "smem-table", "codebook", "hbm-table"))
    ap.add_argument("--kernel", default="auto", choices=("auto", "warp", "cta", "split"))
    ap.add_argument("--opt", action="append", default=[], help="bang_options field=value (e.g. row_prefetch=0)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    k = 10

    import torch
    import torch.distributed as dist
    if world > 1:
        torch.cuda.set_device(local) if torch.cuda.is_available() else None
        import datetime
        # rank 0 builds the artifacts (minutes at C3) while the others wait
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo",
                                init_method="env://", timeout=datetime.timedelta(minutes=45))
    if args.impl == "reference" and rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    from paper_2401_11324_b200 import GraphSearcher, _lib, set_device
    from paper_2401_11324_b200.tools.bench_data import (CLUSTER_SCALE, CONFIGS, EXACT_KNN_LIMIT, HOST_GRAPH_CONFIGS,
                                                        PARTITIONED, THROUGHPUT_CONFIGS, build_artifacts)
    set_device(local)
    thr_only = args.config in THROUGHPUT_CONFIGS
    nq_cfg = 1_000 if args.config == "C1" else (THROUGHPUT_CONFIGS[args.config] if thr_only
                                                 else CONFIGS[args.config])[1]
    ref_world = 1 if args.impl == "reference" else world
    nq_total = nq_cfg * ref_world if args.scaling == "weak" else nq_cfg
    if args.config == "C1":
        art = load_c1_reference(log)
    elif world > 1 and args.impl == "b200":
        # one build per box: rank 0 writes the memory-mapped cache, the others map it
        cache = args.cache or "/tmp/bang_bench_cache"
        if rank == 0:
            art = build_artifacts(args.config, seed=0, nq_total=nq_total, cache_dir=cache, log=log)
        dist.barrier()
        if rank != 0:
            art = build_artifacts(args.config, seed=0, nq_total=nq_total, cache_dir=cache, log=log,
                                  load_only=True)
    else:
        art = build_artifacts(args.config, seed=0, nq_total=nq_total, cache_dir=args.cache or None, log=log)
    # this rank's contiguous query range (sharding.shard_range)
    per = -(-art["queries"].shape[0] // ref_world)
    lo, hi = min(rank * per, art["queries"].shape[0]), min((rank + 1) * per, art["queries"].shape[0])
    queries = np.ascontiguousarray(art["queries"][lo:hi], np.float32)
    gt = None if thr_only else np.asarray(art["gt_ids"][lo:hi])
    nq = queries.shape[0]
    # throughput shapes and C4: graph + vectors in pinned host memory
    mode = "pipelined" if thr_only or args.config in HOST_GRAPH_CONFIGS else "in_memory"
    meta = art["meta"]
    t_fixed = args.t or (meta["t"] if thr_only else 0)
    config = {"workload": args.config, "desc": meta["desc"], "n": meta["n"], "dim": meta["dim"],
              "vectors": meta["dtype"], "R": meta["R"], "m": meta["m"], "k": k,
              "queries_total": int(art["queries"].shape[0]), "queries_per_gpu": nq,
              "bloom_entries": args.bloom, "mode": mode,
              "graph": ("the reference's own VamanaBuilder(R=32, L=64, sigma=1.2) graph" if args.config == "C1" else
                        "seeded random 64-regular graph (no self-loops) in pinned, mapped host memory"
                        if thr_only else
                        "GPU kNN(2R) + RobustPrune(1.2) + reverse edges (tools/graph_build.py)"
                        if meta["n"] <= EXACT_KNN_LIMIT else
                        f"partitioned build (tools/graph_build.build_graph_partitioned: {PARTITIONED[args.config]}): "
                        "per partition IVF kNN(2R) + RobustPrune(1.2) + reverse edges + search-based Vamana "
                        "passes; merged by RobustPrune over each point's partition lists"
                        if args.config in PARTITIONED else
                        "GPU IVF kNN(2R) + RobustPrune(1.2) + reverse edges, then search-based Vamana "
                        "passes (t=128, 128, 200) with this search (tools/graph_build.py)"),
              "cluster_scale": CLUSTER_SCALE.get(args.config, 1.0),
              "l2": "flushed between steps (256 MiB memset outside the step events)",
              "parallelism": f"query-sharded x{ref_world}, index replicated, no collective"}

    if args.impl == "reference":
        # The reference's CPU path = the oracle port, on ALL host threads; the
        # operating point is chosen by the oracle's own recall (no GPU code on
        # this path; the artifacts themselves were built on the GPU).
        def cpu_search(t):
            r, _, _ = cpu_oracle_run(art, queries, t, k, args.bloom)
            return r["ids"], r["iterations"]
        t_sel, sweep = select_t(cpu_search, queries, gt, args.target_recall, k, t_fixed)
        res, sec, cores = cpu_oracle_run(art, queries, t_sel, k, args.bloom)
        # each step a bounded sample: at most ~15 s of CPU work
        n_s = int(min(nq, max(64, nq * 15.0 / max(sec, 1e-9))))
        for _ in range(max(0, args.warmup - 1)):
            cpu_oracle_run(art, queries[:min(n_s, 256)], t_sel, k, args.bloom)
        vals = []
        for _ in range(args.steps):
            _, dt, _ = cpu_oracle_run(art, queries[:n_s], t_sel, k, args.bloom)
            vals.append(n_s / dt)
        v = float(np.mean(vals))
        rec = recall(res["ids"], gt, k)
        metric_name = (f"queries/sec, throughput only ({args.config}, t={t_sel}, no recall)" if thr_only
                       else f"queries/sec at recall@10>=0.9 ({args.config})")
        sample = f"first {n_s} of the {nq} benchmark queries per step, t={t_sel}, k={k}, {cores} host threads"
        out = {"impl": "reference", "metric": metric_name,
               "value": round(v, 2), "unit": "queries/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(1000.0 * n_s / v, 3),
               "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
               "data": "synthetic (seeded Gaussian mixture)", "config": dict(config, t=t_sel),
               "recall_at_10": None if rec is None else round(rec, 4), "t_sweep": sweep,
               "cpu_baseline": {"value": round(v, 2), "unit": "queries/s", "cores": cores,
                                "kind": "port", "sample": sample},
               "e2e": {"value": round(v, 2), "unit": "queries/s", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0}}
        if args.config == "C1":
            out["reference_numpy_qps_here"] = {
                str(t): round(float(art["ref"][f"t{t}_reference_qps"]), 1) for t in art["ref"]["t_values"]}
        print(json.dumps(out), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return

    searcher = GraphSearcher(k=k, t=max(T_SWEEP), mode=mode, bloom_entries=args.bloom, batch_size=max(nq, 1))
    searcher.fit(art["base"], graph=art["graph"], codebook=art["codebook"], codes=art["codes"])
    tuning = {}
    for kv in args.opt:
        key, val = kv.split("=", 1)
        tuning[key] = int(val)
    searcher.set_adc_variant(args.variant).set_kernel(args.kernel, **tuning)

    # ---- worklist size at recall >= target (the metric's operating point)
    def gpu_search(t):
        searcher.t = t
        r = searcher.search(queries)
        return r.ids, r.iterations
    t_sel, sweep = select_t(gpu_search, queries, gt, args.target_recall, k, t_fixed)
    if world > 1:
        tt = torch.tensor([t_sel], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_sel = int(tt.item())
    searcher.t = t_sel
    config["t"] = t_sel
    log(f"[bench] rank {rank}: t={t_sel} sweep={sweep}")
    metric_name = (f"queries/sec, throughput only ({args.config}, t={t_sel}, no recall)" if thr_only
                   else f"queries/sec at recall@10>=0.9 ({args.config})")

    # ---- device-resident timing (value)
    flags = searcher._flags()
    if args.phases:
        flags |= _lib.PROFILE_PHASES
    dev = torch.device("cuda", local)
    dq = torch.from_numpy(queries.copy()).to(dev)
    d_ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    d_dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
    d_it = torch.empty((nq,), dtype=torch.int32, device=dev)
    d_short = torch.empty((nq,), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    # a dedicated stream: the legacy default stream's handle is 0, which the
    # C-ABI reads as "the handle's own stream"
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    h = searcher.index_.handle
    L = _lib.lib()

    def device_step():
        _lib.check(L.bang_search_device(h, _lib.ptr(dq), nq, k, t_sel, args.bloom, flags, _lib.ptr(d_ids),
                                        _lib.ptr(d_dists), _lib.ptr(d_it), _lib.ptr(d_short),
                                        _lib.stream_ptr(stream)), "bang_search_device")

    warm = 1 if args.profile else max(3, args.warmup)
    steps = 1 if args.profile else args.steps
    for _ in range(warm):
        flush.zero_()
        device_step()
        _lib.check(L.bang_sync_status(h))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    kern_ms, stats = [], []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(steps):
            flush.zero_()
            ev[i][0].record(stream)
            device_step()
            ev[i][1].record(stream)
            _lib.check(L.bang_sync_status(h))  # synchronises; outside the events
            st = searcher.index_.stats()
            kern_ms.append(st["kernel_ms"])
            stats.append(st)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(step_ms))
    tmax = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    total_ms = float(tmax.item())
    nq_all = int(art["queries"].shape[0]) if world > 1 else nq
    value = nq_all * steps / (total_ms / 1000.0)
    ids_dev = d_ids.cpu().numpy()
    rec_dev = recall(ids_dev, gt, k)

    if args.profile:
        log(f"[bench] profile step: {step_ms} ms, stats {stats[-1]}")
        return

    # ---- end to end through the public API (pinned host queries)
    qpin = torch.empty(queries.shape, dtype=torch.float32, pin_memory=True)
    qpin.copy_(torch.from_numpy(queries))
    qhost = qpin.numpy()
    e2e_s = []
    res = None
    for i in range(warm + steps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        res = searcher.search(qhost)
        dt = time.perf_counter() - t0
        if i >= warm:
            e2e_s.append(dt)
    e2e_tot = torch.tensor([float(sum(e2e_s))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_tot, op=dist.ReduceOp.MAX)
    e2e_value = nq_all * steps / float(e2e_tot.item())
    rec_e2e = recall(res.ids, gt, k)
    assert np.array_equal(res.ids, ids_dev), "device-resident and end-to-end paths disagree"
    h2d = nq * meta["dim"] * 4
    d2h = nq * (k * 8 + 4 + 1 + 1 + 8 + 8) + 8 + 4 * int(res.iterations.sum())

    # ---- parity at the operating point: the CPU oracle on this rank's whole
    # batch at t_sel, bit-exact (its time is also the CPU baseline)
    parity, cpu = None, None
    if not args.no_parity:
        threads = max(1, (os.cpu_count() or 1) // world)
        want, sec, cores = cpu_oracle_run(art, queries, t_sel, k, args.bloom, threads=threads)
        parity = dict(parity_check(res, want), t=t_sel, kernel="bang::" + _lib.KERNELS.get(stats[-1]["kernel"], "?"))
        if args.config == "C1" and t_sel in meta["reference_outputs"]:
            g = meta["reference_outputs"][t_sel]
            ref = dict(ids=g[f"t{t_sel}_ids"], dists=g[f"t{t_sel}_dists"], iterations=g[f"t{t_sel}_iterations"],
                       short=g[f"t{t_sel}_short"],
                       visit_logs=[g[f"t{t_sel}_log_ids"][a:b] for a, b in
                                   zip(g[f"t{t_sel}_log_offsets"][:-1], g[f"t{t_sel}_log_offsets"][1:])])
            parity["vs_reference_outputs"] = parity_check(res, ref)
        if rank == 0 and not args.no_cpu_baseline:
            cpu = {"value": round(nq / sec, 2), "unit": "queries/s", "cores": cores, "kind": "port",
                   "seconds": round(sec, 3), "queries": nq,
                   "sample": f"all {nq} benchmark queries of rank 0 at t={t_sel}, k={k}, {cores} host threads "
                             f"(OpenMP over queries); the same run is the parity check"}
        if parity["mismatches"]:
            log(f"[bench] PARITY FAILURE: {parity}")
    elif rank == 0 and not args.no_cpu_baseline:
        n_s = min(nq, 2000)
        _, sec, cores = cpu_oracle_run(art, queries[:n_s], t_sel, k, args.bloom)
        cpu = {"value": round(n_s / sec, 2), "unit": "queries/s", "cores": cores, "kind": "port",
               "seconds": round(sec, 3), "queries": n_s,
               "sample": f"first {n_s} benchmark queries at t={t_sel}, k={k}, {cores} host threads"}

    # ---- roofline of the fused search kernel
    peak, peak_kind = measured_peaks()
    s_last = stats[-1]
    avg_kern_ms = float(np.mean(kern_ms))
    achieved = s_last["algorithmic_bytes"] / (avg_kern_ms / 1000.0) / 1e9
    kname = _lib.KERNELS.get(s_last.get("kernel", 0), "?")
    traffic, traffic_note = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(f"{args.config}/{kname}")
            if tr and tr.get("t") == t_sel:
                traffic = tr["dram_bytes_per_launch"]
                traffic_note = f"ncu capture at t={t_sel}: {tr.get('source', '')}"
            elif tr and tr.get("iterations"):
                # the capture's DRAM bytes per query-iteration x this launch's iterations
                traffic = int(round(tr["dram_bytes_per_launch"] / tr["iterations"] * s_last["iterations"]))
                traffic_note = (f"scaled from the ncu capture at t={tr['t']} ({tr['dram_bytes_per_launch']} B over "
                                f"{tr['iterations']} iterations) to this launch's {s_last['iterations']} iterations")
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_note,
                "peak_kind": peak_kind, "kernel": "bang::" + kname, "kernel_ms": round(avg_kern_ms, 4),
                "algorithmic_bytes": s_last["algorithmic_bytes"],
                "bytes_formula": "SURVEY 8(d): I(4R+4) + 20 P + F(m+12) + C(d elem + 12) + nq(4d + 8k)",
                "adc_bytes": s_last["adc_bytes"],
                "adc_gbs": round(s_last["adc_bytes"] / (avg_kern_ms / 1000.0) / 1e9, 1)}

    if mode == "pipelined":
        # host-resident graph (mode="pipelined", C4 and C4r): rows and re-rank vectors
        # cross PCIe; the bound is the measured zero-copy read rate of random
        # rows of the same size (bang_host_read_bandwidth, mode 1)
        import ctypes
        R, d = meta["R"], meta["dim"]
        elem = 1 if meta["dtype"] == "u8" else 4
        row_b = 4 * (R + 4) if R % 4 == 0 else 4 * R
        host_bytes = s_last["iterations"] * row_b + s_last["rerank_cands"] * d * elem
        gbs = ctypes.c_double()
        _lib.check(_lib.lib().bang_host_read_bandwidth(local, 1 << 30, 1, (row_b + 15) // 16 * 16, ctypes.byref(gbs)),
                   "bang_host_read_bandwidth")
        stream_gbs = ctypes.c_double()
        _lib.check(_lib.lib().bang_host_read_bandwidth(local, 1 << 30, 0, 16, ctypes.byref(stream_gbs)),
                   "bang_host_read_bandwidth")
        host_ach = host_bytes / (avg_kern_ms / 1000.0) / 1e9
        roofline["hbm_bound"] = {k2: roofline[k2] for k2 in ("achieved", "peak", "frac")}
        roofline.update({"bound": "pcie", "achieved": round(host_ach, 2), "peak": round(gbs.value, 2),
                         "frac": round(host_ach / gbs.value, 4), "peak_kind": "measured",
                         "peak_source": f"bang_host_read_bandwidth: random {(row_b + 15) // 16 * 16}-byte rows of "
                                        f"pinned mapped host memory (1 GiB), one warp per row",
                         "pcie_stream_gbs": round(stream_gbs.value, 2),
                         "host_bytes": int(host_bytes),
                         "host_bytes_formula": f"I x {row_b} (row with [deg,0,0,0] header) + C x {d * elem} "
                                               f"(re-rank vectors)"})

    # ---- kernel 3 on its own (north_star "ADC kernel HBM GB/s vs peak",
    # SURVEY.md 8(d)): every (query, neighbour) probe of this benchmark's
    # searches, grouped by query, through bang_adc_pairs_device
    adc_k = adc_pairs_roofline(searcher, art, queries, res, dev, stream, flush, peak, peak_kind, warm)

    out = {"metric": metric_name, "value": round(value, 1),
           "unit": "queries/s", "n_gpus": world, "steps": steps, "warmup": warm,
           "ms_per_step": round(total_ms / steps, 4), "higher_is_better": True, "scaling": args.scaling,
           "vs_baseline": None, "dtype": "f32 (u8 codes; f32 ADC sums, f64 re-rank)",
           "data": "synthetic (seeded Gaussian mixture, random-init artifacts built on GPU)",
           "config": config, "recall_at_10": None if rec_e2e is None else round(rec_e2e, 4),
           "recall_device_path": None if rec_dev is None else round(rec_dev, 4),
           "t_sweep": sweep, "parity": parity,
           "e2e": {"value": round(e2e_value, 1), "unit": "queries/s", "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h, "ms_per_step": round(1000 * float(e2e_tot.item()) / steps, 3)},
           "gpu_launches": 2 * steps + (1 if s_last["adc_variant"] == 1 else 0) * steps,
           "roofline": roofline, "adc_kernel": adc_k, "cpu_baseline": cpu,
           "clocks": clk.summary(), "options": searcher.index_.options(),
           "search_stats": {kk: s_last[kk] for kk in ("iterations", "probes", "fresh", "rerank_cands", "slots",
                                                      "warps_per_cta", "ctas", "adc_variant", "retries",
                                                      "kernel")},
           "step_ms": [round(x, 4) for x in step_ms]}
    if args.phases:
        pc = s_last["phase_cycles"]
        it = max(1, s_last["iterations"])
        if s_last.get("kernel") == 8:  # search_split_kernel: row thread 0 / list thread 0 per hop
            prof = searcher.index_.options().get("profile", 0)
            names = {2: ["row_ids", "bloom_words", "pre_bar", "adc", "unused", "coll_bar", "row_end"],
                     3: ["compact", "sort", "merge_reads", "merge_writes", "list_end", "head_won_frac",
                         "survivors_per_hop"]}.get(
                prof, ["row_chain", "list_step", "row_wait_at_hop_barrier", "list_wait_at_hop_barrier"])
            out["phase_cycles_per_iteration"] = {nm: round(pc[i] / it, 3) for i, nm in enumerate(names)}
            out["phase_cycles_per_iteration"]["prologue_epilogue_per_query"] = round(pc[7] / max(1, nq), 1)
        elif s_last.get("kernel") == 2:  # search_cta_kernel: thread 0's cycles
            names = ["bloom_load", "zero_sync", "adc_reduce", "coll_sync", "winner_prefetch", "sort", "merge"]
            out["phase_cycles_per_iteration"] = {nm: round(pc[i] / it, 1) for i, nm in enumerate(names)}
            out["phase_cycles_per_iteration"]["epilogue_per_query"] = round(pc[7] / max(1, nq), 1)
        else:
            names = ["adj_wait", "expand", "bloom_issue", "adc", "bloom_resolve", "sort_eager_prefetch", "merge"]
            out["phase_cycles_per_iteration"] = {nm: round(pc[i] / it, 1) for i, nm in enumerate(names)}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    if parity is not None and parity["mismatches"]:
        sys.exit(3)


if __name__ == "__main__":
    main()
