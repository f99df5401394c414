// bang_search_cta.cuh -- the fused search with one CTA per query (the
// paper's organisation) and the per-query distance table
// in shared memory.  Specialised for 16-byte code rows (m = 16*MV).
//
// Thread i serves neighbour slot j = i/2 of the expanded node's adjacency
// row, half h = i%2:
//   * Bloom: h = 0 hashes/probes slot p1, h = 1 slot p2 (bloom.py:37-42);
//     the pair exchanges its bits with one shuffle;
//   * ADC: h = 0 sums subspaces [0, m/2), h = 1 gathers [m/2, m) and continues
//     the sequential f32 sum from the partner's partial (engine.py:99-105);
//   * sort/merge/re-rank: all threads, barriers between read and write phases.
// Semantics are those of search_kernel / SURVEY.md 8(a0), bit for bit.
//
// Bloom summary (see bang_device.cuh): one smem bit per filter word; words
// first written by this query are zeroed before any atomic touches them --
// across warps, so a CTA barrier separates the zeroing stores from the
// atomics.
#pragma once

#include "bang_kernels.cuh"

namespace bang {

struct CtaMisc {
    unsigned long long wmin[8];  // per-warp survivor minimum
    int wcnt[8];                 // per-warp survivor count
    int wfresh[8];               // per-warp fresh count
    long long qi;
    int hpos;
    int coll;
    unsigned long long head;
    unsigned long long ph[8];  // phase profiler: thread 0's cycles per phase
    long long t_ph;
};
static_assert(sizeof(CtaMisc) <= 256, "CtaMisc must fit its 256-byte smem slot");

// Kernel 5 with the visited rows staged through shared memory: the CTA copies
// a chunk of rows with coalesced 16-byte loads (one PCIe read request per
// 128 B when the vectors live in pinned, mapped host memory, instead of one
// per 4-byte word), then each thread sums its row exactly as exact_sq_dist
// does on the original (engine.py:48-51; same arithmetic, same order).
template <int NT>
__device__ __forceinline__ void rerank_staged(const SearchParams &p, const int32_t *log, int iters,
                                              const float *s_q, uint8_t *stage, int stage_bytes,
                                              uint64_t *rr) {
    const int tid = threadIdx.x;
    const int dim = p.dim, dtype = p.vec_dtype;  // (registers: the stores below may alias p)
    const int rb = dim * (dtype == kVecF32 ? 4 : 1);  // a multiple of 16 (caller)
    const int upr = rb / 16;
    const int ch = stage_bytes / rb;
    const uint8_t *vec = static_cast<const uint8_t *>(p.vectors);
    for (int base = 0; base < iters; base += ch) {
        const int nr = min(ch, iters - base);
        // the rows' 16-byte pieces by cp.async (no register round trip); the
        // log reads of 8 pieces are in flight together, so a chunk costs a few
        // L2 round trips and one HBM round trip, not one of each per piece
#pragma unroll 8
        for (int u = tid; u < nr * upr; u += NT) {
            const int r = u / upr, c = u - r * upr;
            const uint32_t node = (uint32_t)__ldcg(log + base + r);
            __pipeline_memcpy_async(stage + 16 * u, vec + (int64_t)node * rb + 16 * c, 16);
        }
        __pipeline_commit();
        __pipeline_wait_prior(0);
        __syncthreads();
        for (int i = tid; i < nr; i += NT) {
            const uint32_t node = (uint32_t)__ldcg(log + base + i);
            rr[base + i] = pack_key(exact_sq_dist(stage, dtype, dim, i, s_q), node);
        }
        __syncthreads();
    }
}

template <int NT, int SUB, int MV, bool HDR>
// HDR: host-mapped rows with a [deg,0,0,0] header (p.row_hdr), fetched by warp 0
// 768/NT CTAs per SM: 6 queries of 128 threads (R <= 64) fit the register file at <= 80 regs;
// at m = 48 the 48 KB table caps residency at 4 per SM, so allow 128 regs
__global__ void __launch_bounds__(NT, (MV == 3 ? 512 : 768) / NT) search_cta_kernel(const SearchParams p) {
    constexpr int NW = NT / 32;
    constexpr int M = 16 * MV;
    constexpr int MH = M / 2;       // subspaces per half
    constexpr int MHW = MH / 4;     // code words (u32) per half
    constexpr int RPAD = NT / 2;    // neighbour slots
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int j = tid >> 1, h = tid & 1;
    const unsigned lt = (1u << lane) - 1u;

    float *s_q = reinterpret_cast<float *>(smem + p.off_q);
    uint64_t *s_wl = reinterpret_cast<uint64_t *>(smem + p.off_wl);
    uint64_t *s_sk = reinterpret_cast<uint64_t *>(smem + p.off_sk);
    uint64_t *s_nk = reinterpret_cast<uint64_t *>(smem + p.off_nk);
    uint8_t *s_fl = smem + p.off_alive;
    uint8_t *s_vis = smem + p.off_vis;
    uint32_t *s_sum = reinterpret_cast<uint32_t *>(smem + p.off_sum);
    float *s_tab = reinterpret_cast<float *>(smem + p.off_tab);
    CtaMisc *s_m = reinterpret_cast<CtaMisc *>(smem + p.off_acc);
    uint32_t *bits = p.bloom + (int64_t)blockIdx.x * p.bloom_stride;
    uint64_t *rr = p.rr_scratch + (int64_t)blockIdx.x * p.log_cap;
    const int t = p.t, R = p.R;
    const uint64_t hseed = h ? kFnvOffsetH2 : kFnvOffset;

    unsigned long long st_iters = 0, st_probes = 0, st_fresh = 0, st_rr = 0;
    // phase profiler (BANG_PROFILE_PHASES): thread 0's SM cycles per phase,
    // kept in shared memory so the option costs no registers
    if (tid == 0)
        for (int i = 0; i < 8; ++i) s_m->ph[i] = 0;
#define BANG_CTA_PHASE(i)                                      \
    if (p.profile && tid == 0) {                               \
        const long long now_ = clock64();                      \
        s_m->ph[i] += (unsigned long long)(now_ - s_m->t_ph);  \
        s_m->t_ph = now_;                                      \
    }

    for (;;) {
        if (tid == 0) s_m->qi = (long long)atomicAdd(p.counters + kCtrNextQuery, 1ull);
        __syncthreads();
        const int64_t qi = s_m->qi;
        if (qi >= p.nq) break;
        const int64_t qid = p.query_map ? (int64_t)p.query_map[qi] : qi;

        for (int i = tid; i < p.dim; i += NT) s_q[i] = __ldg(p.queries + qid * p.dim + i);
        for (int i = tid; i < p.sum_words; i += NT) s_sum[i] = 0u;
        for (int i = tid; i < t; i += NT) s_vis[i] = 0;
        if (p.bloom_clear) {
            // the filter starts empty: whole-sector stores keep its lines
            // complete in L2, so the fetch-or atomics and word loads of this
            // query hit L2 instead of filling partially written sectors
            uint4 *b4 = reinterpret_cast<uint4 *>(bits);
            const int n4 = (int)(p.bloom_stride >> 2);
            for (int i = tid; i < n4; i += NT) __stcg(b4 + i, make_uint4(0u, 0u, 0u, 0u));
        }
        __syncthreads();
        // kernel 1 for this query into shared memory (pq.py:284-296)
        for (int idx = tid; idx < M * 256; idx += NT) {
            const int s = idx >> 8, c = idx & 255;
            float e;
            if constexpr (SUB == 4) {
                e = table_entry4(*reinterpret_cast<const float4 *>(s_q + s * 4),
                                 __ldg(reinterpret_cast<const float4 *>(p.centroids) + s * 256 + c));
            } else if constexpr (SUB == 2) {
                e = table_entry2(*reinterpret_cast<const float2 *>(s_q + s * 2),
                                 __ldg(reinterpret_cast<const float2 *>(p.centroids) + s * 256 + c));
            } else {
                const int off = __ldg(p.sub_off + s), sz = __ldg(p.sub_size + s);
                const float *src = p.centroids + (int64_t)off * 256 + c * sz;
                float dd = __fsub_rn(s_q[off], __ldg(src));
                float acc = __fmul_rn(dd, dd);
                for (int q = 1; q < sz; ++q) {
                    dd = __fsub_rn(s_q[off + q], __ldg(src + q));
                    acc = __fadd_rn(acc, __fmul_rn(dd, dd));
                }
                e = acc;
            }
            s_tab[idx] = e;
        }
        if (tid == 0) {  // the medoid in the filter (engine.py:127-128)
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
        __syncthreads();
        if (tid == 0) {  // worklist = [key(ADC(medoid), medoid)] (engine.py:118-125)
            const uint8_t *row = p.codes + (int64_t)p.medoid * p.code_stride;
            float acc = 0.0f;
            for (int s = 0; s < M; ++s) acc = __fadd_rn(acc, s_tab[s * 256 + __ldg(row + s)]);
            s_wl[0] = pack_key(acc, (uint32_t)p.medoid);
        }
        int cnt = 1, upos = 0;
        uint32_t u = (uint32_t)p.medoid;
        int deg = p.deg[u];
        uint32_t id = j < R ? (uint32_t)p.adj[(int64_t)u * p.adj_stride + j] : 0u;
        int32_t *log = p.visit_log + (p.query_map ? qi : qid) * p.log_cap;
        int iters = 0;
        __syncthreads();

        for (;;) {
            if (p.profile && tid == 0) s_m->t_ph = clock64();
            // ---- expand u (engine.py:163-178); warp 0 finds the next unvisited
            // entry after u (the eager "head")
            if (warp == 0) {
                if (lane == 0) {
                    if (p.debug && key_id(s_wl[upos]) != u) atomicAdd(p.counters + kCtrDebugFail, 1ull);
                    s_vis[upos] = 1;
                    if (iters < p.log_cap) log[iters] = (int32_t)u;
                }
                __syncwarp();
                const int hp = first_unvisited(s_vis, upos + 1, cnt);
                if (lane == 0) {
                    s_m->hpos = hp;
                    s_m->head = hp < cnt ? s_wl[hp] : kSentinel;
                }
            }
            ++iters;
            st_probes += deg;
            const bool valid = j < deg;
            // ---- this half's code bytes, in flight with the Bloom word
            uint32_t cw[MHW];
            if (valid) {
                const uint32_t *row = reinterpret_cast<const uint32_t *>(p.codes + (int64_t)id * p.code_stride) + h * MHW;
                if constexpr (MHW == 4) {
                    const uint4 v = __ldg(reinterpret_cast<const uint4 *>(row));
                    cw[0] = v.x; cw[1] = v.y; cw[2] = v.z; cw[3] = v.w;
                } else {
#pragma unroll
                    for (int q = 0; q < MHW; q += 2) {
                        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(row + q));
                        cw[q] = v.x;
                        cw[q + 1] = v.y;
                    }
                }
            }
            // ---- kernel 2: Bloom test of this half's slot (pre-state)
            uint32_t ps = 0, word = 0;
            bool init = true;
            if (valid) {
                ps = mod_z(fnv1a(id, hseed), p.geom);
                init = sum_get(s_sum, ps >> 5);
                if (init) word = __ldcg(bits + (ps >> 5));
            }
            const uint32_t mybit = (word >> (ps & 31)) & 1u;
            if (p.profile) asm volatile("" ::"r"(mybit), "r"(cw[0]));
            BANG_CTA_PHASE(0)
            const uint32_t pbit = __shfl_xor_sync(kFull, mybit, 1);
            const uint32_t pps = __shfl_xor_sync(kFull, ps, 1);
            bool fresh = valid && !(mybit && pbit);
            // words first written by this query: zero + summary, then (after
            // the barrier) the fetch-or atomics
            if (fresh && !init) {
                if (!p.bloom_clear) __stcg(bits + (ps >> 5), 0u);
                sum_set(s_sum, ps >> 5);
            }
            __syncthreads();  // zeroing stores (any warp) before any atomic; publishes head
            BANG_CTA_PHASE(1)
            uint32_t old = 0;
            const bool do_atom = fresh && !(h == 1 && pps == ps);
            if (do_atom) old = atomicOr(bits + (ps >> 5), 1u << (ps & 31));
            const uint64_t thr = cnt == t ? s_wl[t - 1] : kSentinel;
            const uint64_t head = s_m->head;
            const int hpos = s_m->hpos;
            uint64_t key = kSentinel;
            bool surv = false;
            uint64_t winner = kSentinel;
            int wid = 0;
            uint32_t nid = 0;
            int ndeg = 0;
            for (int pass = 0; pass < 2; ++pass) {
                // ---- kernel 3: ADC, the two halves chained (engine.py:188-199)
                float e[MH];
                if (fresh) {
#pragma unroll
                    for (int q = 0; q < MH; ++q) {
                        const int s = h * MH + q;
                        e[q] = s_tab[s * 256 + ((cw[q >> 2] >> ((q & 3) * 8)) & 0xFFu)];
                    }
                }
                float acc = 0.0f;
                if (fresh && h == 0) {
#pragma unroll
                    for (int q = 0; q < MH; ++q) acc = __fadd_rn(acc, e[q]);
                }
                const float part = __shfl_xor_sync(kFull, acc, 1);
                key = kSentinel;
                if (fresh && h == 1) {
                    acc = part;
#pragma unroll
                    for (int q = 0; q < MH; ++q) acc = __fadd_rn(acc, e[q]);
                    key = pack_key(acc, id);
                }
                surv = h == 1 && fresh && key < thr;  // ranks >= t are truncated (engine.py:213)
                const uint64_t wm = warp_min_u64(surv ? key : kSentinel);
                const unsigned sb = __ballot_sync(kFull, surv);
                const unsigned fb = __ballot_sync(kFull, fresh && h == 1);
                // Bloom collision check (fetch-or results) folded into the barrier
                const uint32_t b = 1u << (ps & 31);
                const bool coll = pass == 0 && do_atom && (old & b) && !(word & b);
                if (lane == 0) {
                    s_m->wmin[warp] = wm;
                    s_m->wcnt[warp] = __popc(sb);
                    s_m->wfresh[warp] = __popc(fb);
                }
                BANG_CTA_PHASE(2)
                const int any_coll = __syncthreads_or(coll);
                BANG_CTA_PHASE(3)
                if (any_coll) {
                    // in-row slot sharing: exact replay of the involved probes
                    // by warp 0 from the pre-state bits (replay_row_warp)
                    uint2 *rec = reinterpret_cast<uint2 *>(s_sk);
                    uint8_t *fl2 = reinterpret_cast<uint8_t *>(s_nk);
                    if (h == 0) rec[j].x = ps;
                    else rec[j].y = ps;
                    const uint32_t bq = 1u << (ps & 31);
                    fl2[2 * j + h] = (uint8_t)((fresh ? 2 : 0) | ((word & bq) ? 4 : 0) | (coll ? 8 : 0));
                    __syncthreads();
                    if (warp == 0) replay_row_warp<RPAD / 32>(rec, fl2, deg, bits, s_fl);
                    __syncthreads();
                    fresh = valid && s_fl[j];
                    continue;  // redo the ADC with the replayed fresh set
                }
                break;
            }
            // ---- eager winner (engine.py:201-205) -> prefetch its row now
            uint64_t best = kSentinel;
            int n = 0, F = 0, woff = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                best = s_m->wmin[w] < best ? s_m->wmin[w] : best;
                if (w < warp) woff += s_m->wcnt[w];
                n += s_m->wcnt[w];
                F += s_m->wfresh[w];
            }
            winner = best < head ? best : head;
            // host-mapped rows: warp 0 fetches [deg | ids] in one coalesced read,
            // staged to smem at the end of the merge (PCIe: few large requests)
            uint4 rowv = make_uint4(0u, 0u, 0u, 0u);
            const int nchunk = (R + 4) >> 2;
            if (winner != kSentinel) {
                wid = (int)key_id(winner);
                if (HDR) {
                    if (warp == 0 && lane < nchunk)
                        rowv = reinterpret_cast<const uint4 *>(p.adj - 4 + (int64_t)wid * p.adj_stride)[lane];
                } else {
                    ndeg = p.deg[wid];
                    nid = j < R ? (uint32_t)p.adj[(int64_t)wid * p.adj_stride + j] : 0u;
                }
            }
            st_fresh += F;
            // ---- survivors -> s_nk (warp-aggregated), sort (kernel 4a)
            const unsigned sball = __ballot_sync(kFull, surv);
            if (surv) s_nk[woff + __popc(sball & lt)] = key;
            __syncthreads();
            BANG_CTA_PHASE(4)
            for (int q = tid; q < n; q += NT) {
                const uint64_t k = s_nk[q];
                int r = 0, i = 0;
                for (; i + 4 <= n; i += 4)
                    r += (s_nk[i] < k) + (s_nk[i + 1] < k) + (s_nk[i + 2] < k) + (s_nk[i + 3] < k);
                for (; i < n; ++i) r += s_nk[i] < k;
                s_sk[r] = k;
            }
            __syncthreads();
            BANG_CTA_PHASE(5)
            // ---- kernel 4b: merge + truncate to t (engine.py:210-215)
            int wpos = t;
            if (winner != kSentinel)
                wpos = winner != head ? lower_bound_u64(s_wl, cnt, winner) : hpos + lower_bound_u64(s_sk, n, head);
            constexpr int MAXCH = 4;  // worklists up to 4*NT entries (checked on the host)
            uint64_t mv[MAXCH];
            uint8_t mvv[MAXCH];
            int mdst[MAXCH];
#pragma unroll
            for (int c = 0; c < MAXCH; ++c) {
                const int i = c * NT + tid;
                mdst[c] = t;
                mv[c] = 0;
                mvv[c] = 0;
                if (n > 0 && i < cnt) {
                    mv[c] = s_wl[i];
                    mvv[c] = s_vis[i];
                    mdst[c] = i + lower_bound_u64(s_sk, n, mv[c]);
                }
            }
            uint64_t sk = 0;
            int spos = t;
            if (tid < n) {
                sk = s_sk[tid];
                spos = tid + lower_bound_u64(s_wl, cnt, sk);
            }
            __syncthreads();  // all reads of the old worklist precede the writes
            if (n > 0) {
#pragma unroll
                for (int c = 0; c < MAXCH; ++c) {
                    if (mdst[c] < t) {
                        s_wl[mdst[c]] = mv[c];
                        s_vis[mdst[c]] = mvv[c];
                    }
                }
                if (spos < t) {
                    s_wl[spos] = sk;
                    s_vis[spos] = 0;
                }
            }
            cnt = min(t, cnt + n);
            if (HDR && winner != kSentinel && warp == 0 && lane < nchunk)
                reinterpret_cast<uint4 *>(smem + p.off_row)[lane] = rowv;
            __syncthreads();
            BANG_CTA_PHASE(6)
            if (HDR && winner != kSentinel) {
                const int32_t *sr = reinterpret_cast<const int32_t *>(smem + p.off_row);
                ndeg = sr[0];
                nid = j < R ? (uint32_t)sr[4 + j] : 0u;
            }
            // ---- converge (engine.py:217-236)
            if (wpos >= t) break;
            upos = wpos;
            if (p.debug && tid == 0 && s_wl[upos] != winner) atomicAdd(p.counters + kCtrDebugFail, 1ull);
            u = (uint32_t)wid;
            deg = ndeg;
            id = nid;
        }
        st_iters += iters;
        if (p.profile && tid == 0) s_m->t_ph = clock64();

        // ---- outputs (engine.py:244-269)
        int32_t *oid = p.out_ids + qid * p.k;
        float *odist = p.out_dists + qid * p.k;
        if (tid == 0) {
            p.out_iters[qid] = iters;
            p.out_wall_ns[qid] = globaltimer_ns() - p.counters[kCtrT0];
        }
        if (p.rerank) {
            if (iters > p.log_cap) {  // visit log truncated: the host re-runs this query
                if (tid == 0) {
                    const unsigned long long at = atomicAdd(p.counters + kCtrOverflow, 1ull);
                    p.overflow_list[at] = (int32_t)qid;
                }
                __syncthreads();
                continue;
            }
            // kernel 5: exact distances of the visit log, then top-k (warp 0)
            __threadfence_block();
            __syncthreads();
            const int rowb = p.dim * (p.vec_dtype == kVecF32 ? 4 : 1);
            if (rowb % 16 == 0 && rowb <= M * 256 * 4) {
                // the table is dead until the next query: stage rows in its place
                rerank_staged<NT>(p, log, iters, s_q, reinterpret_cast<uint8_t *>(s_tab), M * 256 * 4, rr);
            } else {
                for (int i = tid; i < iters; i += NT) {
                    const uint32_t node = (uint32_t)__ldcg(log + i);
                    rr[i] = pack_key(exact_sq_dist(p.vectors, p.vec_dtype, p.dim, node, s_q), node);
                }
            }
            st_rr += (tid == 0) ? iters : 0;
            __threadfence_block();
            __syncthreads();
            if (warp == 0) {
                warp_topk_write(rr, iters, p.k, oid, odist);
                if (lane == 0) p.out_short[qid] = iters < p.k;
            }
        } else {
            if (p.log_cap < iters && tid == 0) {
                const unsigned long long at = atomicAdd(p.counters + kCtrOverflow, 1ull);
                p.overflow_list[at] = (int32_t)qid;
            }
            for (int q = tid; q < p.k; q += NT) {
                if (q < cnt) {
                    oid[q] = (int32_t)key_id(s_wl[q]);
                    odist[q] = key_dist(s_wl[q]);
                } else {
                    oid[q] = -1;
                    odist[q] = __int_as_float(0x7f800000);
                }
            }
            if (tid == 0) p.out_short[qid] = cnt < p.k;
        }
        __syncthreads();
        BANG_CTA_PHASE(7)
    }
#undef BANG_CTA_PHASE
    if (p.profile && tid == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) atomicAdd(p.counters + kCtrPhase0 + i, s_m->ph[i]);
    }
    if (tid == 0) {
        atomicAdd(p.counters + kCtrIterations, st_iters);
        atomicAdd(p.counters + kCtrRerank, st_rr);
    }
    if (lane == 0) {
        // probes/fresh were accumulated uniformly by every thread: count once per CTA
        if (warp == 0) {
            atomicAdd(p.counters + kCtrProbes, st_probes);
            atomicAdd(p.counters + kCtrFresh, st_fresh);
        }
    }
}

}  // namespace bang
