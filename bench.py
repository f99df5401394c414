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
         host threads) on a bounded sample of the same queries.
Multi-GPU (torchrun): each rank searches its own 10K-query shard against a
replicated index (weak scaling); no collective on the search path.
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


def cpu_oracle_qps(art, t, k, bloom, budget_s=12.0, max_q=None):
    """CPU oracle (C port of the reference path, OpenMP over queries) on a
    bounded sample of the benchmark queries."""
    from oracle import oracle as O
    O.build()
    cores = os.cpu_count() or 1
    q = art["queries"]
    g = art["graph"]
    cb = art["codebook"]
    kw = dict(centroids=cb.centroids, sub_sizes=cb.subspace_sizes, codes=art["codes"].codes,
              adjacency=g.adjacency, degrees=g.degrees, medoid=g.medoid, vectors=art["base"], k=k, t=t,
              bloom_entries=bloom, threads=cores)
    probe = min(q.shape[0], 8 * cores)
    t0 = time.perf_counter()
    O.search(q[:probe], **kw)
    per_q = (time.perf_counter() - t0) / probe
    n = int(min(q.shape[0], max(probe, budget_s / max(per_q, 1e-9))))
    if max_q:
        n = min(n, max_q)
    t0 = time.perf_counter()
    res = O.search(q[:n], **kw)
    dt = time.perf_counter() - t0
    return dict(value=n / dt, unit="queries/s", cores=cores, kind="port", seconds=dt, queries=n,
                sample=f"first {n} of the {q.shape[0]} benchmark queries, t={t}, k={k}, all {cores} host "
                       f"threads (OpenMP over queries)"), res


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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--config", default=os.environ.get("BANG_BENCH_CONFIG", "C3"))
    ap.add_argument("--t", type=int, default=0, help="fixed worklist size (default: recall sweep)")
    ap.add_argument("--target-recall", type=float, default=0.9)
    ap.add_argument("--bloom", type=int, default=399_887)
    ap.add_argument("--cache", default=os.environ.get("BANG_BENCH_CACHE", "/tmp/bang_bench_cache"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="1 warm step + 1 step for ncu; no baselines")
    ap.add_argument("--phases", action="store_true", help="per-phase cycle profile (diagnostic)")
    ap.add_argument("--variant", default="auto", choices=("auto", "smem-table", "smem-table-warp", "smem-table-generic", "codebook", "hbm-table", "pool", "smem-table-nofat", "fat", "pipelined-rows"))
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
    from paper_2401_11324_b200.tools.bench_data import CONFIGS, EXACT_KNN_LIMIT, build_artifacts
    set_device(local)
    from paper_2401_11324_b200.tools.bench_data import THROUGHPUT_CONFIGS
    thr_only = args.config in THROUGHPUT_CONFIGS
    nq = (THROUGHPUT_CONFIGS[args.config] if thr_only else CONFIGS[args.config])[1]
    # each rank owns its own nq-query shard (weak scaling)
    if world > 1:
        # one build per box: rank 0 writes the memory-mapped cache, the others map it
        cache = args.cache or "/tmp/bang_bench_cache"
        if rank == 0:
            art = build_artifacts(args.config, seed=0, nq_total=nq * world, cache_dir=cache, log=log)
        dist.barrier()
        if rank != 0:
            art = build_artifacts(args.config, seed=0, nq_total=nq * world, cache_dir=cache, log=log,
                                  load_only=True)
    else:
        art = build_artifacts(args.config, seed=0, nq_total=nq * world, cache_dir=args.cache or None, log=log)
    lo, hi = rank * nq, (rank + 1) * nq
    shard = dict(art)
    shard["queries"] = art["queries"][lo:hi]
    shard["gt_ids"] = None if thr_only else art["gt_ids"][lo:hi]
    mode = "pipelined" if thr_only else "in_memory"  # throughput shapes: graph in pinned host memory
    meta = art["meta"]
    searcher = GraphSearcher(k=k, t=max(T_SWEEP), mode=mode, bloom_entries=args.bloom,
                             batch_size=nq)
    if args.variant == "fat":
        os.environ["BANG_FAT_ROWS"] = "1"  # search_fat_kernel needs the fat rows built at load
    searcher.fit(art["base"], graph=art["graph"], codebook=art["codebook"], codes=art["codes"])
    searcher.set_adc_variant("auto" if args.variant == "fat" else args.variant)

    # ---- worklist size at recall >= target (the metric's operating point)
    sweep = []
    t_sel = args.t or (meta["t"] if thr_only else 0)
    if not t_sel:
        for t in T_SWEEP:
            searcher.t = t
            res = searcher.search(shard["queries"])
            r = recall(res.ids, shard["gt_ids"], k)
            sweep.append({"t": t, "recall": round(r, 4), "mean_iters": float(res.iterations.mean())})
            if r >= args.target_recall:
                t_sel = t
                break
        if not t_sel:
            t_sel = T_SWEEP[-1]
        elif len(sweep) > 1:
            # the operating point at unit granularity: bisect (t_prev, t_sel]
            # for the smallest t whose recall still meets the target
            lo, hi = sweep[-2]["t"], t_sel
            while hi - lo > 1:
                mid = (lo + hi) // 2
                searcher.t = mid
                res = searcher.search(shard["queries"])
                r = recall(res.ids, shard["gt_ids"], k)
                sweep.append({"t": mid, "recall": round(r, 4), "mean_iters": float(res.iterations.mean())})
                if r >= args.target_recall:
                    hi = mid
                else:
                    lo = mid
            t_sel = hi
    if world > 1:
        tt = torch.tensor([t_sel], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_sel = int(tt.item())
    searcher.t = t_sel
    log(f"[bench] rank {rank}: t={t_sel} sweep={sweep}")

    config = {"workload": args.config, "desc": meta["desc"], "n": meta["n"], "dim": meta["dim"],
              "vectors": meta["dtype"], "R": meta["R"], "m": meta["m"], "k": k, "t": t_sel,
              "queries_per_gpu": nq, "bloom_entries": args.bloom, "mode": mode,
              "graph": ("seeded random 64-regular graph (no self-loops) in pinned, mapped host memory"
                        if thr_only else
                        "GPU kNN(2R) + RobustPrune(1.2) + reverse edges (tools/graph_build.py)"
                        if meta["n"] <= EXACT_KNN_LIMIT else
                        "GPU IVF kNN(2R) + RobustPrune(1.2) + reverse edges, then search-based Vamana "
                        "passes (t=128, 128, 200) with this search (tools/graph_build.py)"),
              "layout": ("random node order" if thr_only else
                         "node ids in k-means partition order (index relabelled at build so graph neighbours "
                         "are near in memory; graph_build.locality_order)" if meta.get("layout") == "partition"
                         else "generator order"),
              "l2": "flushed between steps (256 MiB memset outside the step events)",
              "parallelism": f"query-sharded x{world}, index replicated, no collective"}

    metric_name = (f"queries/sec, throughput only ({args.config}, t={t_sel}, no recall)" if thr_only
                   else f"queries/sec at recall@10>=0.9 ({args.config})")
    if args.impl == "reference":
        cpu, res = cpu_oracle_qps(art, t_sel, k, args.bloom, budget_s=max(5.0, 60.0 / max(1, args.steps)))
        steps = []
        for _ in range(args.steps):
            c, _ = cpu_oracle_qps(art, t_sel, k, args.bloom, budget_s=max(5.0, 60.0 / max(1, args.steps)),
                                  max_q=cpu["queries"])
            steps.append(c["value"])
        v = float(np.mean(steps))
        out = {"impl": "reference", "metric": metric_name,
               "value": round(v, 2), "unit": "queries/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(1000.0 * cpu["queries"] / v, 3),
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
               "data": "synthetic (seeded Gaussian mixture)", "config": config,
               "cpu_baseline": {"value": round(v, 2), "unit": "queries/s", "cores": cpu["cores"],
                                "kind": "port", "sample": cpu["sample"]},
               "e2e": {"value": round(v, 2), "unit": "queries/s", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0}}
        print(json.dumps(out), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- device-resident timing (value)
    flags = _lib.RERANK | searcher._ADC_FLAGS["auto" if args.variant == "fat" else args.variant]
    if args.phases:
        flags |= _lib.PROFILE_PHASES
    dev = torch.device("cuda", local)
    dq = torch.from_numpy(np.ascontiguousarray(shard["queries"], np.float32)).to(dev)
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
    value = nq * world * steps / (total_ms / 1000.0)
    ids_dev = d_ids.cpu().numpy()
    rec_dev = recall(ids_dev, shard["gt_ids"], k)

    if args.profile:
        log(f"[bench] profile step: {step_ms} ms, stats {stats[-1]}")
        return

    # ---- end to end through the public API (pinned host queries)
    qpin = torch.empty(shard["queries"].shape, dtype=torch.float32, pin_memory=True)
    qpin.copy_(torch.from_numpy(np.ascontiguousarray(shard["queries"], np.float32)))
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
    e2e_value = nq * world * steps / float(e2e_tot.item())
    rec_e2e = recall(res.ids, shard["gt_ids"], k)
    assert np.array_equal(res.ids, ids_dev), "device-resident and end-to-end paths disagree"
    h2d = nq * meta["dim"] * 4
    d2h = nq * (k * 8 + 4 + 1 + 1 + 8 + 8) + 8 + 4 * int(res.iterations.sum())

    # ---- roofline of the fused search kernel
    peak, peak_kind = measured_peaks()
    s_last = stats[-1]
    avg_kern_ms = float(np.mean(kern_ms))
    achieved = s_last["algorithmic_bytes"] / (avg_kern_ms / 1000.0) / 1e9
    traffic, traffic_note = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            kname = _lib.KERNELS.get(s_last.get("kernel", 0), "?")
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
                "peak_kind": peak_kind,
                "kernel": "bang::" + _lib.KERNELS.get(s_last.get("kernel", 0), "?"), "kernel_ms": round(avg_kern_ms, 4),
                "algorithmic_bytes": s_last["algorithmic_bytes"],
                "adc_bytes": s_last["adc_bytes"],
                "adc_gbs": round(s_last["adc_bytes"] / (avg_kern_ms / 1000.0) / 1e9, 1)}

    # ---- kernel 3 on its own (north_star "ADC kernel HBM GB/s vs peak",
    # SURVEY.md 8(d)): every (query, neighbour) probe of this benchmark's
    # searches, grouped by query, through bang_adc_pairs_device
    adc_k = adc_pairs_roofline(searcher, art, shard["queries"], res, dev, stream, flush, peak, peak_kind, warm)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu, _ = cpu_oracle_qps(art, t_sel, k, args.bloom)
        cpu = {kk: (round(v, 2) if isinstance(v, float) else v) for kk, v in cpu.items()}

    out = {"metric": metric_name, "value": round(value, 1),
           "unit": "queries/s", "n_gpus": world, "steps": steps, "warmup": warm,
           "ms_per_step": round(total_ms / steps, 4), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32 (u8 codes; f32 ADC sums, f64 re-rank)",
           "data": "synthetic (seeded Gaussian mixture, random-init artifacts built on GPU)",
           "config": config, "recall_at_10": None if rec_e2e is None else round(rec_e2e, 4),
           "recall_device_path": None if rec_dev is None else round(rec_dev, 4),
           "t_sweep": sweep,
           "e2e": {"value": round(e2e_value, 1), "unit": "queries/s", "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h, "ms_per_step": round(1000 * float(e2e_tot.item()) / steps, 3)},
           "gpu_launches": 2 * steps + (1 if s_last["adc_variant"] == 1 else 0) * steps,
           "roofline": roofline, "adc_kernel": adc_k, "cpu_baseline": cpu,
           "clocks": clk.summary(),
           "search_stats": {kk: s_last[kk] for kk in ("iterations", "probes", "fresh", "rerank_cands", "slots",
                                                      "warps_per_cta", "ctas", "adc_variant", "retries",
                                                      "kernel")},
           "step_ms": [round(x, 4) for x in step_ms]}
    if args.phases:
        pc = s_last["phase_cycles"]
        it = max(1, s_last["iterations"])
        if s_last["warps_per_cta"] == 24 and s_last["adc_variant"] == 0:  # search_pool_kernel
            names = ["issue_expand", "bloom_wait_t0", "bloom_barrier", "zeroing", "atomics_adc_t0",
                     "adc_barrier", "replay_owner", "loop_barrier"]
            out["phase_cycles_per_pool_iteration"] = {
                nm: round(pc[i] / max(1, s_last["iterations"] / max(1, s_last["slots"])) / max(1, s_last["ctas"]), 1)
                for i, nm in enumerate(names)}
        elif s_last.get("kernel") == 6:  # search_pf_kernel: thread 32's cycles, slot 1 = warp 0's prefetch
            names = ["bloom_test", "prefetch_warp0", "adc_reduce", "coll_sync", "survivors_sync", "sort",
                     "merge_and_final_sync"]
            out["phase_cycles_per_iteration"] = {nm: round(pc[i] / it, 1) for i, nm in enumerate(names)}
            out["phase_cycles_per_iteration"]["prologue_epilogue_per_query"] = round(pc[7] / max(1, nq), 1)
        elif s_last["slots"] == s_last["ctas"]:  # search_cta_kernel: thread 0's cycles
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


if __name__ == "__main__":
    main()
