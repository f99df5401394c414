// bang_kernels.cuh -- sm_100a kernels of the BANG search path.
//
//   search_kernel          the fused persistent batched search (kernels 2-5
//                          + eager prefetch in one kernel, one warp per query)
//   pq_table_kernel        kernel 1, build_pq_dist_table   (pq.py:284-319)
//   bloom_bank_kernel      kernel 2, filter_and_set        (bloom.py:124-163)
//   adc_kernel             kernel 3, _pq_point_dists+pack  (engine.py:99-105)
//   sort_rows_kernel       kernel 4a, merge_sort_rows      (kernels.py:94-109)
//   merge_rows_kernel      kernel 4b, merge_rows           (kernels.py:68-87)
//   worklist_update_kernel kernel 4, engine step           (engine.py:201-217)
//   rerank_kernel          kernel 5, re-rank               (engine.py:244-262)
//   exact_dists_kernel     exact_sq_dists                  (engine.py:48-51)
#pragma once

#include "bang_device.cuh"

#include <cuda_pipeline.h>

namespace bang {

// counters[] slots of the fused kernel
enum Counter {
    kCtrNextQuery = 0,
    kCtrIterations = 1,
    kCtrProbes = 2,
    kCtrFresh = 3,
    kCtrRerank = 4,
    kCtrOverflow = 5,
    kCtrDebugFail = 6,
    kCtrT0 = 7,
    kCtrPhase0 = 8,  // 8 slots of per-phase SM cycles (BANG_PROFILE_PHASES)
    kCtrNonFinite = 16,  // bang_search: non-finite query values seen on the device
    kCtrCount = 17,
};

// 24 warps x 32 lanes: leaves ptxas 80 registers per thread; shared memory
// already caps the CTA near 24 warps at d = 128.
constexpr int kMaxSearchThreads = 768;

struct SearchParams {
    // index (HBM, or host-mapped for the graph/vectors)
    const uint8_t *codes;
    const float *centroids;  // concat (256, sub_s) f32 over s
    const int32_t *sub_off;  // m (dimension offsets)
    const int32_t *sub_size; // m
    const float *table;      // (nq_map, m, 256) for kAdcGlobalTable, indexed by query id
    const int32_t *adj;      // (n, R) int32, -1 padded
    const int32_t *deg;      // (n,)
    const void *vectors;     // (n, dim) f32/u8/i8
    // batch
    const float *queries;       // (nq_total, dim)
    const int32_t *query_map;   // optional: queries to search this pass
    int64_t nq;                 // queries this pass
    // outputs (indexed by query id)
    int32_t *out_ids;
    float *out_dists;
    int32_t *out_iters;
    uint8_t *out_short;
    uint64_t *out_wall_ns;
    int32_t *visit_log;  // (nq_total, log_cap)
    int64_t log_cap;
    uint64_t *rr_scratch;  // (slots, log_cap) re-rank keys
    int32_t *overflow_list;
    // per-slot Bloom filters
    uint32_t *bloom;
    int64_t bloom_stride;  // u32 words per slot (multiple of 4)
    BloomGeom geom;
    uint32_t medoid_p1, medoid_p2;
    unsigned long long *counters;
    // shapes
    int32_t m, dim, R, medoid, k, t, vec_dtype, adc_variant, rerank, debug, profile;
    int32_t smem_shared_bytes, per_warp_bytes;
    int32_t off_q, off_wl, off_sk, off_nk, off_fid, off_acc, off_alive, off_vis, off_sum, off_tab;  // warp region
    int32_t sum_words;  // u32 words of the Bloom summary (1 bit per filter word)
    int32_t off_dup;    // search_split_kernel: staged code rows / replay records
    // adjacency row i starts at adj + i * adj_stride.  row_hdr: host-mapped
    // rows carry a 16-byte header [deg, 0, 0, 0] at adj - 4 so one coalesced
    // read fetches degree + ids (search_cta_kernel stages it at off_row)
    int64_t adj_stride;
    int32_t row_hdr, off_row;
    // search_cta_kernel: clear the slot's filter with whole-line stores at
    // query start (else words are zeroed on first touch; bang_options.bloom_clear)
    int32_t bloom_clear;
    // search_split_kernel: L2 prefetch of the next head's adjacency row, a
    // candidate for the next winner (bang_options.row_prefetch)
    int32_t row_prefetch;
    // graph + vectors in pinned, mapped host memory (mode="pipelined")
    int32_t host_graph;
    // search_split_kernel: the row keys (double-buffered) at off_code
    int32_t off_code;
    // search_split_kernel: the head's row ids staged by the list warps
    // (bang_options.head_row)
    int32_t off_hrow, head_row;
    // code row stride in bytes (m, or m rounded up to 64 B for m = 48:
    // one DRAM burst per gathered row)
    int32_t code_stride;
    // search_split_kernel (bang_options.bloom_direct): per node, its degree
    // with bit 31 set when two distinct probes of its row share a Bloom slot
    // at this z; rows without it take their pre-state bits from the
    // fetch-or.  Read in place of deg (one load).  nullptr: off
    const int32_t *deg_share;
};

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}


// Top-k of unique keys keys[0, L) (global, written by this warp) into
// out_ids/out_dists; k rounds of a warp-wide min above the last pick.
__device__ __forceinline__ void warp_topk_write(const uint64_t *keys, int64_t L, int k,
                                                int32_t *out_ids, float *out_dists) {
    const int lane = (int)lane_id();
    uint64_t last = 0;
    for (int j = 0; j < k; ++j) {
        uint64_t local = kSentinel;
        if (j < L) {
            for (int64_t i = lane; i < L; i += 32) {
                const uint64_t v = __ldcg(reinterpret_cast<const unsigned long long *>(keys) + i);
                if ((j == 0 || v > last) && v < local) local = v;
            }
        }
        const uint64_t sel = warp_min_u64(local);
        if (lane == 0) {
            if (sel != kSentinel) {
                out_ids[j] = (int32_t)key_id(sel);
                out_dists[j] = key_dist(sel);
            } else {
                out_ids[j] = -1;
                out_dists[j] = __int_as_float(0x7f800000);
            }
        }
        last = sel;
    }
}

// Staged ADC of the fresh neighbours s_fid[0, F) with survivor filtering
// (keys < thr; thr = wl[t-1] when the worklist is full, else SENTINEL):
// survivors' exact keys are compacted into s_nk; returns their count.
template <int SUB, int MV>
__device__ __forceinline__ int adc_survivors(const SearchParams &p, const float *s_cb,
                                             const int *s_off, const int *s_sz,
                                             const float *s_q, int64_t qid,
                                             const uint32_t *s_fid, int F, float *s_acc,
                                             uint8_t *s_alive, uint64_t thr, uint64_t *s_nk,
                                             const float *s_tab) {
    const int lane = (int)lane_id();
    const unsigned lt = (1u << lane) - 1u;
    if (p.adc_variant == kAdcExact) {
        int n = 0;
        for (int base = 0; base < F; base += 32) {
            const int a = base + lane;
            uint64_t key = kSentinel;
            if (a < F) {
                const uint32_t node = s_fid[a];
                key = pack_key(exact_sq_dist(p.vectors, p.vec_dtype, p.dim, node, s_q), node);
            }
            const bool keep = a < F && key < thr;
            const unsigned bal = __ballot_sync(kFull, keep);
            if (keep) s_nk[n + __popc(bal & lt)] = key;
            n += __popc(bal);
        }
        __syncwarp();
        return n;
    }
    const float thr_d = thr == kSentinel ? __int_as_float(0x7f800000) : key_dist(thr);
    const float *trow = p.adc_variant == kAdcSmemTable ? s_tab : p.table + qid * (int64_t)p.m * 256;
    const int m = p.m;
    int n_alive = F;
    for (int s0 = 0; s0 < m && n_alive > 0; s0 += 8) {
        const int ns = min(8, m - s0);
        const bool last = s0 + 8 >= m;
        int n_keep = 0;
        for (int base = 0; base < n_alive; base += 32) {
            const int a = base + lane;
            bool keep = false;
            uint64_t key = 0;
            int j = 0;
            if (a < n_alive) {
                j = s0 == 0 ? a : s_alive[a];
                const uint32_t node = s_fid[j];
                float acc = s0 == 0 ? 0.0f : s_acc[j];
                const uint64_t c8 = load_code8<(MV > 0)>(p.codes + (int64_t)node * p.code_stride, s0, ns);
                if (p.adc_variant == kAdcSmemCodebook)
                    acc = adc_cb_stage<SUB>(acc, s_cb, s_q, s_off, s_sz, s0, ns, c8);
                else
                    acc = adc_tab_stage(acc, trow, s0, ns, c8);
                if (last) {
                    key = pack_key(acc, node);
                    keep = key < thr;
                } else {
                    keep = !(acc > thr_d);
                    s_acc[j] = acc;
                }
            }
            const unsigned bal = __ballot_sync(kFull, keep);
            __syncwarp();  // this round's s_alive reads precede the compaction writes
            if (keep) {
                const int pos = n_keep + __popc(bal & lt);
                if (last) s_nk[pos] = key;
                else s_alive[pos] = (uint8_t)j;
            }
            n_keep += __popc(bal);
        }
        __syncwarp();
        n_alive = n_keep;
        if (last) return n_alive;
    }
    return 0;
}

// 16-byte-code fast path of kernel 3 (m = 16*MV, 16-subspace stages).
// Stage A runs in the lane that owns each probe (codes c0 prefetched with
// the Bloom words); survivors (partial sum <= thr) are compacted into
// s_fid/s_acc and the remaining stages load the next 16 code bytes of the
// survivors only.  Survivor keys (< thr) end up compacted in s_nk.
template <int NPL, int SUB, int MV>
__device__ __forceinline__ int adc_fast_path(const SearchParams &p, const float *s_cb,
                                             const float *s_q, int64_t qid,
                                             const uint32_t (&ids)[NPL], const bool (&fresh)[NPL],
                                             const uint4 (&c0)[NPL], uint64_t thr, uint32_t *s_fid,
                                             float *s_acc, uint64_t *s_nk, const float *s_tab,
                                             int *F_out) {
    const int lane = (int)lane_id();
    const unsigned lt = (1u << lane) - 1u;
    const float thr_d = thr == kSentinel ? __int_as_float(0x7f800000) : key_dist(thr);
    const float *trow = p.adc_variant == kAdcSmemTable ? s_tab : p.table + qid * (int64_t)p.m * 256;
    const bool cb = p.adc_variant == kAdcSmemCodebook;
    int F = 0, n_alive = 0;
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
        bool keep = false;
        float acc = 0.0f;
        uint64_t key = 0;
        if (fresh[k]) {
            acc = cb ? adc_cb_stage16<SUB>(0.0f, s_cb, s_q, 0, c0[k]) : adc_tab_stage16(0.0f, trow, 0, c0[k]);
            if (MV == 1) {
                key = pack_key(acc, ids[k]);
                keep = key < thr;
            } else {
                keep = !(acc > thr_d);
            }
        }
        F += __popc(__ballot_sync(kFull, fresh[k]));
        const unsigned bal = __ballot_sync(kFull, keep);
        if (keep) {
            const int pos = n_alive + __popc(bal & lt);
            if (MV == 1) {
                s_nk[pos] = key;
            } else {
                s_fid[pos] = ids[k];
                s_acc[pos] = acc;
            }
        }
        n_alive += __popc(bal);
    }
    *F_out = F;
    __syncwarp();
#pragma unroll
    for (int st = 1; st < MV; ++st) {
        const bool last = st == MV - 1;
        int n_keep = 0;
        for (int base = 0; base < n_alive; base += 32) {
            const int a = base + lane;
            bool keep = false;
            uint64_t key = 0;
            uint32_t node = 0;
            float acc = 0.0f;
            if (a < n_alive) {
                node = s_fid[a];
                acc = s_acc[a];
                const uint4 cv = __ldg(reinterpret_cast<const uint4 *>(p.codes + (int64_t)node * p.code_stride) + st);
                acc = cb ? adc_cb_stage16<SUB>(acc, s_cb, s_q, 16 * st, cv) : adc_tab_stage16(acc, trow, 16 * st, cv);
                if (last) {
                    key = pack_key(acc, node);
                    keep = key < thr;
                } else {
                    keep = !(acc > thr_d);
                }
            }
            const unsigned bal = __ballot_sync(kFull, keep);
            __syncwarp();  // this round's reads precede the compaction writes
            if (keep) {
                const int pos = n_keep + __popc(bal & lt);
                if (last) {
                    s_nk[pos] = key;
                } else {
                    s_fid[pos] = node;
                    s_acc[pos] = acc;
                }
            }
            n_keep += __popc(bal);
        }
        __syncwarp();
        n_alive = n_keep;
    }
    return n_alive;
}

// -------------------------------------------------------------------------
// The fused persistent search kernel.  One warp owns one query at a time
// (dynamic fetch from an atomic counter, so stragglers never idle an SM);
// per-query state: worklist + visited flags + query vector + Bloom summary
// in shared memory, Bloom words in HBM/L2, the next candidate's adjacency
// row in registers.  Per iteration (engine.py:152-236):
//   expand u -> Bloom test-and-set of u's neighbours (kernel 2; atomics in
//   flight) -> staged ADC of the fresh ones with survivor filtering
//   (kernel 3) -> resolve the Bloom atomics -> sort survivors, eager winner
//   = min(best survivor, first unvisited) and the winner's adjacency row is
//   loaded NOW ("one hop ahead") -> merge + truncate to t
//   (kernel 4) -> converged when the winner is gone or truncated.
// At convergence the warp re-ranks its visit log with exact distances
// (kernel 5) and writes the query's outputs.
// -------------------------------------------------------------------------
template <int NPL, int SUB, int MV>
__global__ void __launch_bounds__(kMaxSearchThreads, 1) search_kernel(const SearchParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = (int)lane_id();
    const int warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const int slot = blockIdx.x * nwarps + warp;

    float *s_cb = reinterpret_cast<float *>(smem);
    int *s_off = nullptr, *s_sz = nullptr;
    if (p.adc_variant == kAdcSmemCodebook) {
        const int n4 = (256 * p.dim) / 4;
        const float4 *src = reinterpret_cast<const float4 *>(p.centroids);
        float4 *dst = reinterpret_cast<float4 *>(s_cb);
        for (int i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = __ldg(src + i);
        s_off = reinterpret_cast<int *>(smem + (size_t)256 * p.dim * 4);
        s_sz = s_off + p.m;
        if (!(SUB > 0 && MV > 0)) {
            for (int i = threadIdx.x; i < p.m; i += blockDim.x) {
                s_off[i] = p.sub_off[i];
                s_sz[i] = p.sub_size[i];
            }
        }
        __syncthreads();
    }
    unsigned char *wbase = smem + p.smem_shared_bytes + (size_t)warp * p.per_warp_bytes;
    float *s_q = reinterpret_cast<float *>(wbase + p.off_q);
    uint64_t *s_wl = reinterpret_cast<uint64_t *>(wbase + p.off_wl);
    uint64_t *s_sk = reinterpret_cast<uint64_t *>(wbase + p.off_sk);
    uint64_t *s_nk = reinterpret_cast<uint64_t *>(wbase + p.off_nk);
    uint32_t *s_fid = reinterpret_cast<uint32_t *>(wbase + p.off_fid);
    float *s_acc = reinterpret_cast<float *>(wbase + p.off_acc);
    uint8_t *s_alive = wbase + p.off_alive;
    uint8_t *s_vis = wbase + p.off_vis;
    uint32_t *s_sum = reinterpret_cast<uint32_t *>(wbase + p.off_sum);
    float *s_tab = reinterpret_cast<float *>(wbase + p.off_tab);
    uint32_t *bits = p.bloom + (int64_t)slot * p.bloom_stride;
    uint64_t *rr = p.rr_scratch + (int64_t)slot * p.log_cap;
    const int t = p.t, R = p.R;

    unsigned long long st_iters = 0, st_probes = 0, st_fresh = 0, st_rr = 0;

    for (;;) {
        int64_t qi = 0;
        if (lane == 0) qi = (int64_t)atomicAdd(p.counters + kCtrNextQuery, 1ull);
        qi = __shfl_sync(kFull, qi, 0);
        if (qi >= p.nq) break;
        const int64_t qid = p.query_map ? (int64_t)p.query_map[qi] : qi;

        // query vector -> smem; empty Bloom summary (the filter words are
        // never cleared: unsummarised words read as 0); vis flags
        for (int j = lane; j < p.dim; j += 32) s_q[j] = __ldg(p.queries + qid * p.dim + j);
        for (int j = lane; j < p.sum_words; j += 32) s_sum[j] = 0u;
        for (int j = lane; j < t; j += 32) s_vis[j] = 0;
        __syncwarp();
        if (p.adc_variant == kAdcSmemTable) {  // kernel 1 for this query, into smem
            build_table_warp<SUB>(s_tab, s_q, p.centroids, p.sub_off, p.sub_size, p.m);
            __syncwarp();
        }
        // medoid in the filter (engine.py:127-128 set_all_rows)
        if (lane == 0) {
            const uint32_t w1 = p.medoid_p1 >> 5, w2 = p.medoid_p2 >> 5;
            const uint32_t b1 = 1u << (p.medoid_p1 & 31), b2 = 1u << (p.medoid_p2 & 31);
            if (w1 == w2) {
                __stcg(bits + w1, b1 | b2);
            } else {
                __stcg(bits + w1, b1);
                __stcg(bits + w2, b2);
            }
            s_sum[w1 >> 5] |= 1u << (w1 & 31);
            s_sum[w2 >> 5] |= 1u << (w2 & 31);
        }
        // worklist = [key(score(medoid), medoid)] (engine.py:118-125)
        float d0 = 0.f;
        if (lane == 0) {
            if (p.adc_variant == kAdcSmemCodebook)
                d0 = adc_codebook<SUB, MV>(s_cb, s_q, s_off, s_sz, p.m, p.codes + (int64_t)p.medoid * p.code_stride);
            else if (p.adc_variant == kAdcGlobalTable)
                d0 = adc_table<MV>(p.table + qid * (int64_t)p.m * 256, p.m, p.codes + (int64_t)p.medoid * p.code_stride);
            else if (p.adc_variant == kAdcSmemTable)
                d0 = adc_table<MV>(s_tab, p.m, p.codes + (int64_t)p.medoid * p.code_stride);
            else
                d0 = exact_sq_dist(p.vectors, p.vec_dtype, p.dim, p.medoid, s_q);
            s_wl[0] = pack_key(d0, (uint32_t)p.medoid);
        }
        __threadfence_block();
        __syncwarp();
        int cnt = 1, upos = 0;
        uint32_t u = (uint32_t)p.medoid;
        uint32_t ids[NPL];
        int deg = p.deg[u];
#pragma unroll
        for (int k = 0; k < NPL; ++k) {
            const int c = lane + 32 * k;
            ids[k] = c < R ? (uint32_t)p.adj[(int64_t)u * p.adj_stride + c] : 0u;
        }
        // log rows follow the pass order when a query map is given (retry pass)
        int32_t *log = p.visit_log + (p.query_map ? qi : qid) * p.log_cap;
        int iters = 0;

        for (;;) {
            // phase profiler (flag BANG_PROFILE_PHASES): SM cycles per phase,
            // summed over warps; the asm makes the wait for the prefetched
            // adjacency row land in phase 0
            long long t_ph = 0;
#define BANG_PHASE(i)                                                               \
    if (p.profile) {                                                                \
        const long long now_ = clock64();                                           \
        if (lane == 0) atomicAdd(p.counters + kCtrPhase0 + (i), (unsigned long long)(now_ - t_ph)); \
        t_ph = now_;                                                                \
    }
            if (p.profile) {
                t_ph = clock64();
                asm volatile("" ::"r"(ids[0]), "r"(deg));
                BANG_PHASE(0)
            }
            // ---- expand u (engine.py:163-178)
            if (p.debug && lane == 0 && key_id(s_wl[upos]) != u)
                atomicAdd(p.counters + kCtrDebugFail, 1ull);
            if (lane == 0) {
                s_vis[upos] = 1;
                if (iters < p.log_cap) log[iters] = (int32_t)u;
            }
            ++iters;
            st_probes += deg;
            // ---- kernel 2: Bloom test-and-set in adjacency order (engine.py:180-186)
            // (16-byte code path: the first 16 code bytes of every neighbour are
            // requested together with the Bloom words, off the critical path)
            uint4 c0[NPL];
            if constexpr (MV > 0) {
#pragma unroll
                for (int k = 0; k < NPL; ++k)
                    if (lane + 32 * k < deg)
                        c0[k] = __ldg(reinterpret_cast<const uint4 *>(p.codes + (int64_t)ids[k] * p.code_stride));
            }
            BANG_PHASE(1)
            BloomRow<NPL> br;
            bloom_issue<NPL>(bits, s_sum, p.geom, ids, deg, br);
            if (p.profile) asm volatile("" ::"r"((int)br.fresh[0]));
            BANG_PHASE(2)
            const uint64_t thr = cnt == t ? s_wl[t - 1] : kSentinel;
            int F = 0, n_s = 0;
            if constexpr (MV > 0) {
                // ---- kernel 3: staged ADC; stage A (subspaces 0-15) in the
                // probe's own lane, later stages on compacted survivors
                if (p.adc_variant != kAdcExact) {
                    n_s = adc_fast_path<NPL, SUB, MV>(p, s_cb, s_q, qid, ids, br.fresh, c0, thr, s_fid, s_acc,
                                                      s_nk, s_tab, &F);
                    BANG_PHASE(3)
                    if (bloom_resolve<NPL>(bits, s_sum, p.geom, ids, deg, br))
                        n_s = adc_fast_path<NPL, SUB, MV>(p, s_cb, s_q, qid, ids, br.fresh, c0, thr, s_fid,
                                                          s_acc, s_nk, s_tab, &F);
                }
            } else {
                for (int pass = 0; pass < 2; ++pass) {
                    // ---- compact the fresh ids (warp-aggregated ballot + popc)
                    F = 0;
#pragma unroll
                    for (int k = 0; k < NPL; ++k) {
                        const unsigned b = __ballot_sync(kFull, br.fresh[k]);
                        if (br.fresh[k]) s_fid[F + __popc(b & ((1u << lane) - 1u))] = ids[k];
                        F += __popc(b);
                    }
                    __syncwarp();
                    // ---- kernel 3: staged ADC of the fresh neighbours (engine.py:188-199)
                    n_s = adc_survivors<SUB, MV>(p, s_cb, s_off, s_sz, s_q, qid, s_fid, F, s_acc, s_alive, thr,
                                                 s_nk, s_tab);
                    // ---- the Bloom atomics' results (collision -> exact replay, redo)
                    if (pass == 0 && !bloom_resolve<NPL>(bits, s_sum, p.geom, ids, deg, br)) break;
                }
            }
            BANG_PHASE(4)
            st_fresh += F;
            // ---- sort survivors; eager winner (engine.py:201-205)
            sort_keys(s_nk, n_s, s_sk);
            const int hpos = first_unvisited(s_vis, upos + 1, cnt);
            const uint64_t head = hpos < cnt ? s_wl[hpos] : kSentinel;
            const uint64_t best = n_s > 0 ? s_sk[0] : kSentinel;
            const uint64_t winner = best < head ? best : head;
            // ---- one-hop-ahead prefetch of the winner's adjacency row
            uint32_t nids[NPL];
            int ndeg = 0;
            if (winner != kSentinel) {
                const uint32_t w = key_id(winner);
                ndeg = p.deg[w];
#pragma unroll
                for (int k = 0; k < NPL; ++k) {
                    const int c = lane + 32 * k;
                    nids[k] = c < R ? (uint32_t)p.adj[(int64_t)w * p.adj_stride + c] : 0u;
                }
            } else {
#pragma unroll
                for (int k = 0; k < NPL; ++k) nids[k] = 0u;
            }
            BANG_PHASE(5)
            // ---- kernel 4: merge + truncate (engine.py:210-215)
            int first = 0;
            const int old_cnt = cnt;
            cnt = merge_sorted(s_wl, s_vis, cnt, t, s_sk, n_s, &first);
            // ---- converge (engine.py:217-236): the winner is the new first
            // unvisited entry unless it was truncated away
            int wpos = t;
            if (winner != kSentinel) {
                if (best < head) wpos = first;
                else wpos = hpos + lower_bound_u64(s_sk, n_s, head);
            }
            (void)old_cnt;
            BANG_PHASE(6)
            if (wpos >= t) break;
            upos = wpos;
            if (p.debug && lane == 0 && s_wl[upos] != winner) atomicAdd(p.counters + kCtrDebugFail, 1ull);
            u = key_id(winner);
            deg = ndeg;
#pragma unroll
            for (int k = 0; k < NPL; ++k) ids[k] = nids[k];
        }
        st_iters += iters;

        // ---- outputs (engine.py:244-269)
        int32_t *oid = p.out_ids + qid * p.k;
        float *odist = p.out_dists + qid * p.k;
        if (lane == 0) {
            p.out_iters[qid] = iters;
            p.out_wall_ns[qid] = globaltimer_ns() - p.counters[kCtrT0];
        }
        if (p.rerank && p.adc_variant != kAdcExact) {
            if (iters > p.log_cap) {  // visit log truncated: the host re-runs this query
                if (lane == 0) {
                    const unsigned long long at = atomicAdd(p.counters + kCtrOverflow, 1ull);
                    p.overflow_list[at] = (int32_t)qid;
                }
                continue;
            }
            // kernel 5: exact distances of the visit log, then top-k
            __syncwarp();
            for (int i = lane; i < iters; i += 32) {
                const uint32_t node = (uint32_t)__ldcg(log + i);
                rr[i] = pack_key(exact_sq_dist(p.vectors, p.vec_dtype, p.dim, node, s_q), node);
            }
            st_rr += iters;
            __threadfence_block();
            __syncwarp();
            warp_topk_write(rr, iters, p.k, oid, odist);
            if (lane == 0) p.out_short[qid] = iters < p.k;
        } else {
            if (p.log_cap < iters && lane == 0) {
                const unsigned long long at = atomicAdd(p.counters + kCtrOverflow, 1ull);
                p.overflow_list[at] = (int32_t)qid;
            }
            for (int j = lane; j < p.k; j += 32) {
                if (j < cnt) {
                    oid[j] = (int32_t)key_id(s_wl[j]);
                    odist[j] = key_dist(s_wl[j]);
                } else {
                    oid[j] = -1;
                    odist[j] = __int_as_float(0x7f800000);
                }
            }
            if (lane == 0) p.out_short[qid] = cnt < p.k;
        }
        __syncwarp();
    }
    if (lane == 0) {
        atomicAdd(p.counters + kCtrIterations, st_iters);
        atomicAdd(p.counters + kCtrProbes, st_probes);
        atomicAdd(p.counters + kCtrFresh, st_fresh);
        atomicAdd(p.counters + kCtrRerank, st_rr);
    }
}

}  // namespace bang
