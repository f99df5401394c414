// bang_search_fat.cuh -- one CTA per query over "fat" adjacency rows.
//
// The CTA-per-query search (bang_search_cta.cuh) spends each iteration in
// three serialized memory waits (profiles/r01/phases_C3_cta.json): the Bloom
// words + PQ code rows of u's neighbours (~2.9K cycles incl. the slowest of
// 128 loads), the Bloom fetch-or round trip consumed by the collision check,
// and the sort/merge.  This kernel removes the first two from the critical
// path:
//
//  * fat rows: node u's row holds its neighbour ids AND their PQ code rows,
//        [ids: R x int32][pad to 16 B][codes: R x m bytes]
//    (HBM: n x 3.3 KB at C3), built once at index load (build_fat_rows_kernel).
//    The eager winner's whole row is fetched one hop ahead in ONE coalesced
//    read that lands during the sort/merge, so the ADC never waits on a
//    dependent code gather (PAPER.md:922-938's prefetch, widened to codes).
//  * speculative ADC: every valid neighbour's distance is computed from the
//    smem table while the Bloom words are in flight; the Bloom result only
//    masks (fresh & key < thr) -- the reference's arithmetic is unchanged.
//  * exact in-row slot sharing in shared memory: each probe's slot is
//    inserted into a 256-entry CAS hash table while the words load; a probe
//    that finds its slot taken is "shared".  Only fresh shared probes can
//    change the sequential test-and-set outcome (bloom.py:134-158), and for
//    those warp 0 replays the involved probes in adjacency order from the
//    pre-state bits already in registers (no L2 round trips).  The Bloom
//    fetch-ors are then fire-and-forget (RED), issued after the survivors
//    are published.
// Semantics are SURVEY.md 8(a0), bit for bit (same table entries, same
// sequential f32 ADC sums, same keys, sort, merge, truncation, re-rank).
#pragma once

#include "bang_search_cta.cuh"

namespace bang {


// One warp per node: ids, then the code rows of its neighbours (m = 16*MV).
__global__ void build_fat_rows_kernel(const int32_t *__restrict__ adj, const int32_t *__restrict__ deg,
                                      const uint8_t *__restrict__ codes, int64_t n, int R, int m,
                                      int code_off, int64_t stride, uint8_t *__restrict__ fat) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int v16 = m / 16;
    for (int64_t u = w; u < n; u += nw) {
        uint8_t *row = fat + u * stride;
        const int d = deg[u];
        for (int j = lane; j < R; j += 32) reinterpret_cast<int32_t *>(row)[j] = adj[u * R + j];
        for (int x = lane; x < d * v16; x += 32) {
            const int j = x / v16, v = x % v16;
            const int64_t nb = adj[u * R + j];
            reinterpret_cast<uint4 *>(row + code_off + (int64_t)j * m)[v] =
                reinterpret_cast<const uint4 *>(codes + nb * m)[v];
        }
    }
}

template <int NT, int SUB, int MV, int MINB>
__global__ void __launch_bounds__(NT, MINB) search_fat_kernel(const SearchParams p) {
    constexpr int NW = NT / 32;
    constexpr int M = 16 * MV;
    constexpr int MH = M / 2;       // subspaces per half
    constexpr int MHW = MH / 4;     // code words (u32) per half
    constexpr int RPAD = NT / 2;    // neighbour slots
    constexpr int NPL = RPAD / 32;  // replay: probes per lane of warp 0
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int j = tid >> 1, h = tid & 1;
    const unsigned lt = (1u << lane) - 1u;

    float *s_q = reinterpret_cast<float *>(smem + p.off_q);
    uint64_t *s_wl = reinterpret_cast<uint64_t *>(smem + p.off_wl);
    uint64_t *s_sk = reinterpret_cast<uint64_t *>(smem + p.off_sk);
    uint64_t *s_nk = reinterpret_cast<uint64_t *>(smem + p.off_nk);
    uint8_t *s_fl = smem + p.off_alive;  // replay records: flags per (probe, half)
    uint8_t *s_vis = smem + p.off_vis;
    uint32_t *s_sum = reinterpret_cast<uint32_t *>(smem + p.off_sum);
    float *s_tab = reinterpret_cast<float *>(smem + p.off_tab);
    uint32_t *s_dup = reinterpret_cast<uint32_t *>(smem + p.off_dup);
    uint8_t *s_tf = smem + p.off_dup + 4 * kDupSlots;  // replay: truly fresh per probe
    CtaMisc *s_m = reinterpret_cast<CtaMisc *>(smem + p.off_acc);
    uint32_t *bits = p.bloom + (int64_t)blockIdx.x * p.bloom_stride;
    uint64_t *rr = p.rr_scratch + (int64_t)blockIdx.x * p.log_cap;
    const int t = p.t, R = p.R;
    const uint64_t hseed = h ? kFnvOffsetH2 : kFnvOffset;
    const int64_t fstride = p.fat_stride;
    const int coff = p.fat_code_off + j * M + h * MH;

    // fat row of node u: this thread's neighbour id and its half of the code
    // row (ld.global.cg: a coherent load, so it is issued where written and
    // lands during the sort/merge instead of being sunk to its first use)
    auto load_row = [&](uint32_t u, uint32_t &id, uint32_t (&cw)[MHW]) {
        const uint8_t *row = p.fat + (int64_t)u * fstride;
        id = 0u;
        if (j < R) {
            id = __ldcg(reinterpret_cast<const unsigned int *>(row) + j);
            if constexpr (MHW == 4) {
                const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(row + coff));
                cw[0] = v.x; cw[1] = v.y; cw[2] = v.z; cw[3] = v.w;
            } else {
#pragma unroll
                for (int q = 0; q < MHW; q += 2) {
                    const uint2 v = __ldcg(reinterpret_cast<const uint2 *>(row + coff) + q / 2);
                    cw[q] = v.x;
                    cw[q + 1] = v.y;
                }
            }
        }
    };

    unsigned long long st_iters = 0, st_probes = 0, st_fresh = 0, st_rr = 0;
    for (int i = tid; i < kDupSlots; i += NT) s_dup[i] = kDupEmpty;

    for (;;) {
        if (tid == 0) s_m->qi = (long long)atomicAdd(p.counters + kCtrNextQuery, 1ull);
        __syncthreads();
        const int64_t qi = s_m->qi;
        if (qi >= p.nq) break;
        const int64_t qid = p.query_map ? (int64_t)p.query_map[qi] : qi;

        for (int i = tid; i < p.dim; i += NT) s_q[i] = __ldg(p.queries + qid * p.dim + i);
        for (int i = tid; i < p.sum_words; i += NT) s_sum[i] = 0u;
        for (int i = tid; i < t; i += NT) s_vis[i] = 0;
        __syncthreads();
        // kernel 1 for this query into shared memory (pq.py:284-296)
        for (int idx = tid; idx < M * 256; idx += NT) {
            const int s = idx >> 8, c = idx & 255;
            float e;
            if constexpr (SUB == 4) {
                e = table_entry4(*reinterpret_cast<const float4 *>(s_q + s * 4),
                                 __ldg(reinterpret_cast<const float4 *>(p.centroids) + s * 256 + c));
            } else {
                e = table_entry2(*reinterpret_cast<const float2 *>(s_q + s * 2),
                                 __ldg(reinterpret_cast<const float2 *>(p.centroids) + s * 256 + c));
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
            const uint8_t *row = p.codes + (int64_t)p.medoid * M;
            float acc = 0.0f;
            for (int s = 0; s < M; ++s) acc = __fadd_rn(acc, s_tab[s * 256 + __ldg(row + s)]);
            s_wl[0] = pack_key(acc, (uint32_t)p.medoid);
        }
        int cnt = 1, upos = 0;
        uint32_t u = (uint32_t)p.medoid;
        int deg = p.deg[u];
        uint32_t id, cw[MHW];
        load_row(u, id, cw);
        int32_t *log = p.visit_log + (p.query_map ? qi : qid) * p.log_cap;
        int iters = 0;
        __syncthreads();

        for (;;) {
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
            // ---- kernel 2, pre-state: this half's slot; the word load flies
            // while the slot is hashed into the row's sharing table and the
            // ADC runs
            uint32_t ps = 0, word = 0;
            bool init = true;
            if (valid) {
                ps = mod_z(fnv1a(id, hseed), p.geom);
                init = sum_get(s_sum, ps >> 5);
                if (init) word = __ldcg(bits + (ps >> 5));
            }
            const uint32_t pps = __shfl_xor_sync(kFull, ps, 1);
            const bool self = h == 1 && pps == ps;  // p1 == p2: one slot, one insert
            bool shared = false;
            int didx = -1;
            if (valid && !self) {
                uint32_t x = (ps * 0x9E3779B1u) >> 24;
                for (;;) {
                    const uint32_t old = atomicCAS(s_dup + x, kDupEmpty, ps);
                    if (old == kDupEmpty) {
                        didx = (int)x;
                        break;
                    }
                    if (old == ps) {
                        shared = true;
                        break;
                    }
                    x = (x + 1) & (kDupSlots - 1);
                }
            }
            // ---- kernel 3: speculative ADC of every neighbour (engine.py:99-105),
            // the two halves chained through a shuffle (sequential f32 sum)
            float e[MH];
            if (valid) {
#pragma unroll
                for (int q = 0; q < MH; ++q) {
                    const int s = h * MH + q;
                    e[q] = s_tab[s * 256 + ((cw[q >> 2] >> ((q & 3) * 8)) & 0xFFu)];
                }
            }
            float acc = 0.0f;
            if (valid && h == 0) {
#pragma unroll
                for (int q = 0; q < MH; ++q) acc = __fadd_rn(acc, e[q]);
            }
            const float part = __shfl_xor_sync(kFull, acc, 1);
            uint64_t key = kSentinel;
            if (valid && h == 1) {
                acc = part;
#pragma unroll
                for (int q = 0; q < MH; ++q) acc = __fadd_rn(acc, e[q]);
                key = pack_key(acc, id);
            }
            const uint64_t thr = cnt == t ? s_wl[t - 1] : kSentinel;
            // ---- the pre-state bits (the word loads land here)
            const uint32_t mybit = (word >> (ps & 31)) & 1u;
            const uint32_t pbit = __shfl_xor_sync(kFull, mybit, 1);
            bool fresh = valid && !(mybit && pbit);
            const bool at_risk = fresh && shared;
            bool surv = h == 1 && fresh && key < thr;  // ranks >= t are truncated (engine.py:213)
            {
                const uint64_t wm = warp_min_u64(surv ? key : kSentinel);
                const unsigned sb = __ballot_sync(kFull, surv);
                const unsigned fb = __ballot_sync(kFull, fresh && h == 1);
                if (lane == 0) {
                    s_m->wmin[warp] = wm;
                    s_m->wcnt[warp] = __popc(sb);
                    s_m->wfresh[warp] = __popc(fb);
                }
            }
            const int any_risk = __syncthreads_or(at_risk);  // B1: all summary reads done
            if (didx >= 0) s_dup[didx] = kDupEmpty;          // every insert of this row is done
            if (any_risk) {
                // ---- rare: in-row slot sharing among fresh probes -> exact
                // replay of the involved probes in adjacency order
                if (h == 0) reinterpret_cast<uint2 *>(s_sk)[j].x = ps;
                else reinterpret_cast<uint2 *>(s_sk)[j].y = ps;
                s_fl[2 * j + h] = (uint8_t)((valid ? 1 : 0) | (fresh ? 2 : 0) | (mybit ? 4 : 0) | (shared ? 8 : 0));
                __syncthreads();
                if (warp == 0) {
                    uint32_t a[NPL], b[NPL];
                    bool pf[NPL], pre1[NPL], pre2[NPL], inv[NPL], tf[NPL], dr[NPL];
#pragma unroll
                    for (int r = 0; r < NPL; ++r) {
                        const int jj = lane + 32 * r;
                        const uint2 v = jj < deg ? reinterpret_cast<const uint2 *>(s_sk)[jj] : make_uint2(0u, 0u);
                        const uint8_t f0 = jj < deg ? s_fl[2 * jj] : 0, f1 = jj < deg ? s_fl[2 * jj + 1] : 0;
                        a[r] = v.x;
                        b[r] = v.y;
                        pf[r] = jj < deg && (f0 & 2);  // presumed fresh (pre-state test)
                        pre1[r] = f0 & 4;
                        pre2[r] = f1 & 4;
                        inv[r] = pf[r] && ((f0 | f1) & 8);
                        tf[r] = dr[r] = false;
                    }
                    // partners of the shared probes
#pragma unroll
                    for (int rc = 0; rc < NPL; ++rc) {
                        unsigned cm = __ballot_sync(kFull, inv[rc]);
                        while (cm) {
                            const int src = __ffs(cm) - 1;
                            cm &= cm - 1;
                            const uint32_t pa = __shfl_sync(kFull, a[rc], src), pb = __shfl_sync(kFull, b[rc], src);
#pragma unroll
                            for (int r = 0; r < NPL; ++r)
                                inv[r] = inv[r] || (pf[r] && (a[r] == pa || a[r] == pb || b[r] == pa || b[r] == pb));
                        }
                    }
                    auto in_set = [&](uint32_t pos) {
                        bool hit = false;
#pragma unroll
                        for (int r = 0; r < NPL; ++r) hit = hit || (tf[r] && (a[r] == pos || b[r] == pos));
                        return __any_sync(kFull, hit);
                    };
                    // sequential test-and-set over the involved probes (bloom.py:110-122)
#pragma unroll
                    for (int r = 0; r < NPL; ++r) {
                        unsigned im = __ballot_sync(kFull, inv[r]);
                        while (im) {
                            const int src = __ffs(im) - 1;
                            im &= im - 1;
                            const uint32_t pa = __shfl_sync(kFull, a[r], src), pb = __shfl_sync(kFull, b[r], src);
                            const bool q1 = __shfl_sync(kFull, (int)pre1[r], src), q2 = __shfl_sync(kFull, (int)pre2[r], src);
                            const bool h1 = q1 || in_set(pa);
                            const bool h2 = q2 || in_set(pb);
                            if (lane == src) {
                                if (!(h1 && h2)) tf[r] = true;
                                else dr[r] = true;
                            }
                        }
                    }
#pragma unroll
                    for (int r = 0; r < NPL; ++r) {
                        const int jj = lane + 32 * r;
                        if (jj < RPAD) s_tf[jj] = (uint8_t)(pf[r] && !dr[r]);
                    }
                }
                __syncthreads();
                fresh = valid && s_tf[j];
                surv = h == 1 && fresh && key < thr;
                const uint64_t wm = warp_min_u64(surv ? key : kSentinel);
                const unsigned sb = __ballot_sync(kFull, surv);
                const unsigned fb = __ballot_sync(kFull, fresh && h == 1);
                if (lane == 0) {
                    s_m->wmin[warp] = wm;
                    s_m->wcnt[warp] = __popc(sb);
                    s_m->wfresh[warp] = __popc(fb);
                }
                __syncthreads();
            }
            // ---- words first written by this query: zero + summary (the
            // fetch-ors follow after the next barrier)
            if (fresh && !init && !self) {
                __stcg(bits + (ps >> 5), 0u);
                sum_set(s_sum, ps >> 5);
            }
            // ---- eager winner (engine.py:201-205) -> fetch its fat row now
            const uint64_t head = s_m->head;
            const int hpos = s_m->hpos;
            uint64_t best = kSentinel;
            int n = 0, F = 0, woff = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                best = s_m->wmin[w] < best ? s_m->wmin[w] : best;
                if (w < warp) woff += s_m->wcnt[w];
                n += s_m->wcnt[w];
                F += s_m->wfresh[w];
            }
            const uint64_t winner = best < head ? best : head;
            uint32_t nid = 0, ncw[MHW];
            int ndeg = 0;
            int wid = 0;
            if (winner != kSentinel) {
                wid = (int)key_id(winner);
                ndeg = p.deg[wid];
                load_row((uint32_t)wid, nid, ncw);
            }
            st_fresh += F;
            // ---- survivors -> s_nk (warp-aggregated)
            const unsigned sball = __ballot_sync(kFull, surv);
            if (surv) s_nk[woff + __popc(sball & lt)] = key;
            __syncthreads();  // B2: zeroing stores before the fetch-ors; survivors published
            // ---- Bloom set of the fresh probes: fire-and-forget (RED)
            if (fresh && !self) atomicOr(bits + (ps >> 5), 1u << (ps & 31));
            // ---- sort survivors (kernel 4a)
            for (int q = tid; q < n; q += NT) {
                const uint64_t k = s_nk[q];
                int r = 0, i = 0;
                for (; i + 4 <= n; i += 4)
                    r += (s_nk[i] < k) + (s_nk[i + 1] < k) + (s_nk[i + 2] < k) + (s_nk[i + 3] < k);
                for (; i < n; ++i) r += s_nk[i] < k;
                s_sk[r] = k;
            }
            __syncthreads();
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
            __syncthreads();
            // ---- converge (engine.py:217-236)
            if (wpos >= t) break;
            upos = wpos;
            if (p.debug && tid == 0 && s_wl[upos] != winner) atomicAdd(p.counters + kCtrDebugFail, 1ull);
            u = (uint32_t)wid;
            deg = ndeg;
            id = nid;
#pragma unroll
            for (int q = 0; q < MHW; ++q) cw[q] = ncw[q];
        }
        st_iters += iters;

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
            for (int i = tid; i < iters; i += NT) {
                const uint32_t node = (uint32_t)__ldcg(log + i);
                rr[i] = pack_key(exact_sq_dist(p.vectors, p.vec_dtype, p.dim, node, s_q), node);
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
    }
    if (tid == 0) {
        atomicAdd(p.counters + kCtrIterations, st_iters);
        atomicAdd(p.counters + kCtrRerank, st_rr);
    }
    if (lane == 0 && warp == 0) {
        // probes/fresh were accumulated uniformly by every thread: count once per CTA
        atomicAdd(p.counters + kCtrProbes, st_probes);
        atomicAdd(p.counters + kCtrFresh, st_fresh);
    }
}

}  // namespace bang
