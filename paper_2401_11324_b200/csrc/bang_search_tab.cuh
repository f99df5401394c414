// bang_search_tab.cuh -- the fused search kernel specialised for the
// per-query shared-memory distance table (ADC variant 3, the paper's layout)
// and 16-byte code rows (m = 16*MV).
//
// Same semantics as search_kernel (engine.py:108-270); the
// iteration is laid out for latency, since only 4-6 queries fit per SM:
//   * the whole code row of every neighbour is requested into registers
//     together with the Bloom words, so the ADC never waits on memory;
//   * the ADC is m table lookups (LDS) + m sequential f32 adds per fresh
//     neighbour, in the lane that owns the probe;
//   * the eager winner is known right after the ADC (warp min over the
//     survivors and the first unvisited entry), so the next adjacency row
//     is requested before the Bloom atomics are resolved and before the
//     survivors are sorted and merged;
//   * sort/merge: independent binary searches, all reads before writes.
#pragma once

#include "bang_kernels.cuh"

namespace bang {

// worklist merge for sorted survivors s_sk[0, n) (n <= 128), t <= 32*MAXCH:
// every wl element and every survivor computes its final rank with an
// independent binary search in the other list, then all are written at once.
template <int MAXCH>
__device__ __forceinline__ int merge_sorted_regs(uint64_t *s_wl, uint8_t *s_vis, int cnt, int t,
                                                 const uint64_t *s_sk, int n) {
    const int lane = (int)lane_id();
    if (n == 0) return cnt;
    uint64_t v[MAXCH];
    uint8_t vv[MAXCH];
    int dst[MAXCH];
#pragma unroll
    for (int c = 0; c < MAXCH; ++c) {
        const int i = c * 32 + lane;
        dst[c] = t;
        v[c] = 0;
        vv[c] = 0;
        if (i < cnt) {
            v[c] = s_wl[i];
            vv[c] = s_vis[i];
        }
    }
#pragma unroll
    for (int c = 0; c < MAXCH; ++c)
        if (c * 32 + lane < cnt) dst[c] = c * 32 + lane + lower_bound_u64(s_sk, n, v[c]);
    int pos[4];
    uint64_t kv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int j = q * 32 + lane;
        pos[q] = t;
        kv[q] = 0;
        if (j < n) {
            kv[q] = s_sk[j];
            pos[q] = j + lower_bound_u64(s_wl, cnt, kv[q]);
        }
    }
    __syncwarp();  // every read above precedes every write below
#pragma unroll
    for (int c = 0; c < MAXCH; ++c) {
        if (dst[c] < t) {
            s_wl[dst[c]] = v[c];
            s_vis[dst[c]] = vv[c];
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (pos[q] < t) {
            s_wl[pos[q]] = kv[q];
            s_vis[pos[q]] = 0;
        }
    }
    __syncwarp();
    return min(t, cnt + n);
}

// rank sort of s_nk[0, n) into s_sk (broadcast reads, 4 in flight)
__device__ __forceinline__ void sort_keys_unrolled(const uint64_t *s_nk, int n, uint64_t *s_sk) {
    const int lane = (int)lane_id();
    for (int j = lane; j < n; j += 32) {
        const uint64_t k = s_nk[j];
        int r = 0;
        int i = 0;
        for (; i + 4 <= n; i += 4) {
            const uint64_t a = s_nk[i], b = s_nk[i + 1], c = s_nk[i + 2], d = s_nk[i + 3];
            r += (a < k) + (b < k) + (c < k) + (d < k);
        }
        for (; i < n; ++i) r += s_nk[i] < k;
        s_sk[r] = k;
    }
    __syncwarp();
}

// sum_{s<m} T[s][code_s] over a register-resident code row (m = 16*MV)
template <int MV>
__device__ __forceinline__ float adc_row_smem(const float *s_tab, const uint4 (&cv)[MV]) {
    float acc = 0.0f;
#pragma unroll
    for (int v = 0; v < MV; ++v) {
        const uint32_t w[4] = {cv[v].x, cv[v].y, cv[v].z, cv[v].w};
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            const int s = v * 16 + b;
            acc = __fadd_rn(acc, s_tab[s * 256 + ((w[b >> 2] >> ((b & 3) * 8)) & 0xFFu)]);
        }
    }
    return acc;
}

template <int NPL, int SUB, int MV>
__global__ void __launch_bounds__(256, 1) search_tab_kernel(const SearchParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = (int)lane_id();
    const int warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const int slot = blockIdx.x * nwarps + warp;
    const unsigned lt = (1u << lane) - 1u;

    unsigned char *wbase = smem + (size_t)warp * p.per_warp_bytes;
    float *s_q = reinterpret_cast<float *>(wbase + p.off_q);
    uint64_t *s_wl = reinterpret_cast<uint64_t *>(wbase + p.off_wl);
    uint64_t *s_sk = reinterpret_cast<uint64_t *>(wbase + p.off_sk);
    uint64_t *s_nk = reinterpret_cast<uint64_t *>(wbase + p.off_nk);
    uint8_t *s_vis = wbase + p.off_vis;
    uint32_t *s_sum = reinterpret_cast<uint32_t *>(wbase + p.off_sum);
    float *s_tab = reinterpret_cast<float *>(wbase + p.off_tab);
    uint32_t *bits = p.bloom + (int64_t)slot * p.bloom_stride;
    uint64_t *rr = p.rr_scratch + (int64_t)slot * p.log_cap;
    const int t = p.t, R = p.R, m = p.m;

    unsigned long long st_iters = 0, st_probes = 0, st_fresh = 0, st_rr = 0;

    for (;;) {
        int64_t qi = 0;
        if (lane == 0) qi = (int64_t)atomicAdd(p.counters + kCtrNextQuery, 1ull);
        qi = __shfl_sync(kFull, qi, 0);
        if (qi >= p.nq) break;
        const int64_t qid = p.query_map ? (int64_t)p.query_map[qi] : qi;

        for (int j = lane; j < p.dim; j += 32) s_q[j] = __ldg(p.queries + qid * p.dim + j);
        for (int j = lane; j < p.sum_words; j += 32) s_sum[j] = 0u;
        for (int j = lane; j < t; j += 32) s_vis[j] = 0;
        __syncwarp();
        // kernel 1 for this query, into shared memory (pq.py:284-296)
        build_table_warp<SUB>(s_tab, s_q, p.centroids, p.sub_off, p.sub_size, m);
        if (lane == 0) {  // the medoid in the filter (engine.py:127-128)
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
        __threadfence_block();
        __syncwarp();
        if (lane == 0) {  // worklist = [key(ADC(medoid), medoid)] (engine.py:118-125)
            uint4 cm[MV];
#pragma unroll
            for (int v = 0; v < MV; ++v)
                cm[v] = __ldg(reinterpret_cast<const uint4 *>(p.codes + (int64_t)p.medoid * m) + v);
            s_wl[0] = pack_key(adc_row_smem<MV>(s_tab, cm), (uint32_t)p.medoid);
        }
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
        int32_t *log = p.visit_log + (p.query_map ? qi : qid) * p.log_cap;
        int iters = 0;

        for (;;) {
            // ---- expand u (engine.py:163-178)
            if (p.debug && lane == 0 && key_id(s_wl[upos]) != u) atomicAdd(p.counters + kCtrDebugFail, 1ull);
            if (lane == 0) {
                s_vis[upos] = 1;
                if (iters < p.log_cap) log[iters] = (int32_t)u;
            }
            ++iters;
            st_probes += deg;
            // ---- the neighbours' code rows, in flight with the Bloom words
            uint4 cv[NPL][MV];
#pragma unroll
            for (int k = 0; k < NPL; ++k)
                if (lane + 32 * k < deg)
#pragma unroll
                    for (int v = 0; v < MV; ++v)
                        cv[k][v] = __ldg(reinterpret_cast<const uint4 *>(p.codes + (int64_t)ids[k] * m) + v);
            // ---- kernel 2: Bloom test-and-set in adjacency order (engine.py:180-186)
            BloomRow<NPL> br;
            bloom_issue<NPL>(bits, s_sum, p.geom, ids, deg, br);
            const uint64_t thr = cnt == t ? s_wl[t - 1] : kSentinel;
            const int hpos = first_unvisited(s_vis, upos + 1, cnt);
            const uint64_t head = hpos < cnt ? s_wl[hpos] : kSentinel;
            uint64_t key[NPL];
            uint64_t winner = kSentinel;
            uint32_t nids[NPL];
            int ndeg = 0;
            for (int pass = 0; pass < 2; ++pass) {
                // ---- kernel 3: ADC of the fresh neighbours (engine.py:188-199)
                uint64_t best = kSentinel;
#pragma unroll
                for (int k = 0; k < NPL; ++k) {
                    key[k] = kSentinel;
                    if (br.fresh[k]) {
                        key[k] = pack_key(adc_row_smem<MV>(s_tab, cv[k]), ids[k]);
                        if (key[k] >= thr) key[k] = kSentinel;  // ranks >= t: truncated
                    }
                    best = key[k] < best ? key[k] : best;
                }
                // ---- eager winner (engine.py:201-205) -> prefetch its row now
                best = warp_min_u64(best);
                const uint64_t w = best < head ? best : head;
                if (pass == 0 || w != winner) {
                    winner = w;
                    if (winner != kSentinel) {
                        const uint32_t wid = key_id(winner);
                        ndeg = p.deg[wid];
#pragma unroll
                        for (int k = 0; k < NPL; ++k) {
                            const int c = lane + 32 * k;
                            nids[k] = c < R ? (uint32_t)p.adj[(int64_t)wid * p.adj_stride + c] : 0u;
                        }
                    }
                }
                // ---- the Bloom atomics' results (collision -> exact replay, redo)
                if (pass == 0 && !bloom_resolve<NPL>(bits, s_sum, p.geom, ids, deg, br)) break;
            }
            int F = 0, n = 0;
#pragma unroll
            for (int k = 0; k < NPL; ++k) {
                F += __popc(__ballot_sync(kFull, br.fresh[k]));
                const bool keep = key[k] != kSentinel;
                const unsigned b = __ballot_sync(kFull, keep);
                if (keep) s_nk[n + __popc(b & lt)] = key[k];
                n += __popc(b);
            }
            st_fresh += F;
            __syncwarp();
            // ---- kernel 4: sort + merge + truncate (engine.py:210-215)
            sort_keys_unrolled(s_nk, n, s_sk);
            int wpos = t;
            if (winner != kSentinel) {  // position of the winner after the merge
                if (winner != head) wpos = lower_bound_u64(s_wl, cnt, winner);  // = s_sk[0]'s slot
                else wpos = hpos + lower_bound_u64(s_sk, n, head);
            }
            if (t <= 256) cnt = merge_sorted_regs<8>(s_wl, s_vis, cnt, t, s_sk, n);
            else {
                int first = 0;
                cnt = merge_sorted(s_wl, s_vis, cnt, t, s_sk, n, &first);
            }
            // ---- converge (engine.py:217-236)
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
        if (p.rerank) {
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
