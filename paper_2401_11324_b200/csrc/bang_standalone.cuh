// bang_standalone.cuh -- the stand-alone per-kernel entry points of
// libbang.so (one reference function each; bang.h "per-kernel entries"),
// compiled only into bang_abi.cu.
#pragma once

#include "bang_kernels.cuh"

namespace bang {

__global__ void record_t0_kernel(unsigned long long *counters) {
    counters[kCtrT0] = globaltimer_ns();
}

// validation.py:17-19 ("contains non-finite values") on the device, over the
// queries bang_search has just uploaded: the host skips its own pass over
// them.  One flag per warp that sees a NaN/inf.
__global__ void check_finite_kernel(const float *__restrict__ x, int64_t count, unsigned long long *counters) {
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(__ldg(x + i));
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicAdd(counters + kCtrNonFinite, 1ull);
}

// Rows with in-row Bloom slot sharing at Bloom size z (bloom.py:135-151's
// "fresh candidates of one row share a slot", taken over ALL probes of the
// row): out[w] = deg[w] | (1 << 31) when two distinct probes among node w's
// first deg[w] neighbours have a slot in common, else deg[w].  A row without
// it behaves identically under batched and sequential test-and-set, and each
// probe's fetch-or returns exactly the pre-state of its own bits.  One warp
// per row; the row's 2*deg slots in shared memory, every lane compares its
// own against all of them.  Built once per (index, z).
constexpr int kShareWarps = 8;
__global__ void __launch_bounds__(32 * kShareWarps) row_share_kernel(const int32_t *__restrict__ adj,
                                                                     int64_t adj_stride,
                                                                     const int32_t *__restrict__ deg,
                                                                     int64_t n, int R, BloomGeom g,
                                                                     int32_t *__restrict__ out) {
    extern __shared__ uint32_t s_slots[];  // [kShareWarps][2R]
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    uint32_t *sl = s_slots + wi * 2 * R;
    for (int64_t w = (int64_t)blockIdx.x * kShareWarps + wi; w < n; w += (int64_t)gridDim.x * kShareWarps) {
        const int dw = deg[w];
        const int d = min(max(dw, 0), R);
        const int32_t *row = adj + w * adj_stride;
        for (int j = lane; j < d; j += 32) {
            const uint32_t id = (uint32_t)row[j];
            sl[2 * j] = mod_z(fnv1a(id, kFnvOffset), g);
            sl[2 * j + 1] = mod_z(fnv1a(id, kFnvOffsetH2), g);
        }
        __syncwarp();
        // branch-free: every lane holds its (up to) four slots in registers
        // and compares them with each broadcast slot of the row (R <= 64;
        // wider rows take the strided loop below)
        bool dup = false;
        if (d <= 64) {
            uint32_t v[4];
            int pa[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int a = lane + 32 * k;
                v[k] = a < 2 * d ? sl[a] : 0xFFFFFFFFu;  // slots are < z < 2^31: never equal
                pa[k] = a >> 1;
            }
#pragma unroll 8
            for (int b = 0; b < 2 * d; ++b) {
                const uint32_t x = sl[b];
                const int pb = b >> 1;
#pragma unroll
                for (int k = 0; k < 4; ++k) dup |= (x == v[k]) & (pb != pa[k]);
            }
        } else {
            for (int a = lane; a < 2 * d; a += 32) {
                const uint32_t v = sl[a];
                for (int b = 0; b < 2 * d; ++b) dup |= (sl[b] == v) & ((b >> 1) != (a >> 1));
            }
        }
        const bool shared = __any_sync(kFull, dup);
        if (lane == 0) out[w] = shared ? (int32_t)((uint32_t)d | 0x80000000u) : d;
        __syncwarp();
    }
}

// -------------------------------------------------------------------------
// Kernel 1 -- build_pq_dist_table (pq.py:284-319).  One CTA per query,
// thread c = centroid c, subspaces in order; each subspace row (1 KB) is
// written coalesced.  Exact f32 op order, no FMA.
// -------------------------------------------------------------------------
__global__ void __launch_bounds__(256) pq_table_kernel(const float *__restrict__ centroids,
                                                       const int32_t *__restrict__ sub_off,
                                                       const int32_t *__restrict__ sub_size,
                                                       int m, int dim,
                                                       const float *__restrict__ queries,
                                                       float *__restrict__ out) {
    extern __shared__ float s_qt[];
    const int64_t q = blockIdx.x;
    for (int j = threadIdx.x; j < dim; j += blockDim.x) s_qt[j] = __ldg(queries + q * dim + j);
    __syncthreads();
    const int c = threadIdx.x;
    float *o = out + q * (int64_t)m * 256;
    for (int s = 0; s < m; ++s) {
        const int off = __ldg(sub_off + s), sz = __ldg(sub_size + s);
        const float *cc = centroids + (int64_t)off * 256 + (int64_t)c * sz;
        float d = __fsub_rn(s_qt[off], __ldg(cc));
        float acc = __fmul_rn(d, d);
        for (int j = 1; j < sz; ++j) {
            d = __fsub_rn(s_qt[off + j], __ldg(cc + j));
            acc = __fadd_rn(acc, __fmul_rn(d, d));
        }
        __stcs(o + s * 256 + c, acc);
    }
}

// -------------------------------------------------------------------------
// Kernel 2 -- BloomFilterBank.filter_and_set (bloom.py:124-163): one warp
// per filter row, the row's probes processed 32 at a time in order.
// -------------------------------------------------------------------------
__global__ void bloom_bank_kernel(uint32_t *bits, int64_t count, int64_t words32, BloomGeom g,
                                  const int64_t *__restrict__ row_off,
                                  const uint32_t *__restrict__ ids, uint8_t *fresh) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= count) return;
    const int lane = (int)lane_id();
    uint32_t *b = bits + row * words32;
    const int64_t lo = row_off[row], hi = row_off[row + 1];
    for (int64_t base = lo; base < hi; base += 32) {
        const int cnt = (int)min((int64_t)32, hi - base);
        uint32_t id[1] = {lane < cnt ? ids[base + lane] : 0u};
        bool fr[1];
        bloom_test_and_set<1>(b, nullptr, g, id, cnt, fr);
        if (lane < cnt) fresh[base + lane] = fr[0] ? 1 : 0;
    }
}

// -------------------------------------------------------------------------
// Kernel 3 -- ADC over (query row, node) pairs (engine.py:99-105) with the
// key pack of engine.py:195-199.  One thread per pair, code row gathered as
// 16-byte vectors when m % 16 == 0.
// -------------------------------------------------------------------------
template <int MV>
__global__ void adc_kernel(const float *__restrict__ table, int m,
                           const uint8_t *__restrict__ codes, const int64_t *__restrict__ qrows,
                           const uint32_t *__restrict__ ids, int64_t n, float *dists,
                           uint64_t *keys) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t node = __ldg(ids + i);
    const float d = adc_table<MV>(table + __ldg(qrows + i) * (int64_t)m * 256, m,
                                  codes + (int64_t)node * m);
    if (dists) dists[i] = d;
    if (keys) keys[i] = pack_key(d, node);
}

// -------------------------------------------------------------------------
// Kernel 4a -- merge_sort_rows (kernels.py:94-109).  One CTA per row; each
// element's stable rank (#less + #equal-before) is its output slot, which
// yields exactly the ascending row for any width.
// -------------------------------------------------------------------------
__global__ void sort_rows_kernel(uint64_t *keys, int w) {
    extern __shared__ uint64_t s_row[];
    uint64_t *row = keys + (int64_t)blockIdx.x * w;
    for (int i = threadIdx.x; i < w; i += blockDim.x) s_row[i] = row[i];
    __syncthreads();
    for (int i = threadIdx.x; i < w; i += blockDim.x) {
        const uint64_t v = s_row[i];
        int r = 0;
        for (int j = 0; j < w; ++j) {
            const uint64_t x = s_row[j];
            r += (x < v) || (x == v && j < i);
        }
        row[r] = v;
    }
}

// Kernel 4b -- merge_rows (kernels.py:68-87): a_i -> i + #{b < a_i};
// b_j -> j + #{a <= b_j} (the reference's rank merge, a first on ties).
__global__ void merge_rows_kernel(const uint64_t *__restrict__ a, const uint8_t *__restrict__ a_pay,
                                  int wa, const uint64_t *__restrict__ b, int wb, uint64_t *out,
                                  uint8_t *out_pay) {
    const int64_t r = blockIdx.x;
    const uint64_t *ar = a + r * wa, *br = b + r * wb;
    uint64_t *o = out + r * (int64_t)(wa + wb);
    uint8_t *op = out_pay ? out_pay + r * (int64_t)(wa + wb) : nullptr;
    for (int i = threadIdx.x; i < wa; i += blockDim.x) {
        const int pos = i + lower_bound_u64(br, wb, ar[i]);
        o[pos] = ar[i];
        if (op) op[pos] = a_pay ? a_pay[r * wa + i] : 0;
    }
    for (int j = threadIdx.x; j < wb; j += blockDim.x) {
        const int pos = j + upper_bound_u64(ar, wa, br[j]);
        o[pos] = br[j];
        if (op) op[pos] = 0;
    }
}

// -------------------------------------------------------------------------
// Kernel 4 (engine step) -- eager pick + sort + merge + truncate + converge
// (engine.py:201-217) per worklist row, one warp per row, through the same
// survivor filter / sort_keys / merge_sorted the fused kernel runs.
// Shared memory per warp: wl keys (t), sorted + unsorted new keys (w each),
// visited flags (t).
// -------------------------------------------------------------------------
__global__ void worklist_update_kernel(uint64_t *wl_keys, uint8_t *wl_vis, int64_t rows, int t,
                                       const uint64_t *__restrict__ new_keys, int w,
                                       uint64_t *winner, uint8_t *done) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = (int)lane_id();
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (row >= rows) return;
    const int a_wl = (t * 8 + 15) & ~15, a_k = (w * 8 + 15) & ~15;
    const int per_warp = a_wl + 2 * a_k + ((t + 15) & ~15);
    unsigned char *base = smem + (size_t)warp * per_warp;
    uint64_t *s_wl = reinterpret_cast<uint64_t *>(base);
    uint64_t *s_sk = reinterpret_cast<uint64_t *>(base + a_wl);
    uint64_t *s_nk = reinterpret_cast<uint64_t *>(base + a_wl + a_k);
    uint8_t *s_vis = base + a_wl + 2 * a_k;
    uint64_t *gw = wl_keys + row * t;
    uint8_t *gv = wl_vis + row * t;
    int cnt = 0;
    for (int b = 0; b < t; b += 32) {
        const int i = b + lane;
        bool real = false;
        if (i < t) {
            s_wl[i] = gw[i];
            s_vis[i] = gv[i];
            real = gw[i] != kSentinel;
        }
        cnt += __popc(__ballot_sync(kFull, real));
    }
    __syncwarp();
    // survivors: non-sentinel new keys that can rank below t
    const uint64_t thr = cnt == t ? s_wl[t - 1] : kSentinel;
    int n = 0;
    uint64_t best_all = kSentinel;
    for (int b = 0; b < w; b += 32) {
        const int i = b + lane;
        const uint64_t v = i < w ? new_keys[row * w + i] : kSentinel;
        best_all = v < best_all ? v : best_all;
        const bool keep = v != kSentinel && v < thr;
        const unsigned m = __ballot_sync(kFull, keep);
        if (keep) s_nk[n + __popc(m & ((1u << lane) - 1u))] = v;
        n += __popc(m);
    }
    best_all = warp_min_u64(best_all);
    __syncwarp();
    sort_keys(s_nk, n, s_sk);
    const int hpos = first_unvisited(s_vis, 0, cnt);
    const uint64_t head = hpos < cnt ? s_wl[hpos] : kSentinel;
    const uint64_t win = best_all < head ? best_all : head;  // engine.py:202-204 (all new keys)
    int first = 0;
    cnt = merge_sorted(s_wl, s_vis, cnt, t, s_sk, n, &first);
    const int upos = first_unvisited(s_vis, 0, cnt);
    for (int i = lane; i < t; i += 32) {
        gw[i] = i < cnt ? s_wl[i] : kSentinel;
        gv[i] = i < cnt ? s_vis[i] : 0;
    }
    if (lane == 0) {
        winner[row] = win;
        done[row] = upos >= cnt ? 1 : 0;
    }
}

// -------------------------------------------------------------------------
// Kernel 5 -- re-rank (engine.py:244-262): one warp per query over its
// candidates; keys staged in `scratch` (same CSR layout).
// -------------------------------------------------------------------------
__global__ void rerank_kernel(const void *vectors, int dtype, int dim,
                              const float *__restrict__ queries, int64_t nq,
                              const int64_t *__restrict__ off, const int32_t *__restrict__ cand,
                              uint64_t *scratch, int k, int32_t *out_ids, float *out_dists,
                              uint8_t *out_short) {
    extern __shared__ float s_qr[];
    const int warp = threadIdx.x >> 5, lane = (int)lane_id();
    const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (q >= nq) return;
    float *sq = s_qr + (size_t)warp * dim;
    for (int j = lane; j < dim; j += 32) sq[j] = queries[q * dim + j];
    __syncwarp();
    const int64_t lo = off[q], L = off[q + 1] - lo;
    for (int64_t i = lane; i < L; i += 32) {
        const uint32_t node = (uint32_t)cand[lo + i];
        scratch[lo + i] = pack_key(exact_sq_dist(vectors, dtype, dim, node, sq), node);
    }
    __threadfence_block();
    __syncwarp();
    warp_topk_write(scratch + lo, L, k, out_ids + q * k, out_dists + q * k);
    if (lane == 0) out_short[q] = L < k;
}

// Visit-log compaction: row r of a (rows, cap) log -> CSR at out + off[dst(r)],
// dst(r) = map ? map[r] : r.  One warp per row.
__global__ void compact_logs_kernel(const int32_t *__restrict__ log, int64_t cap, int64_t rows,
                                    const int32_t *__restrict__ map, const int64_t *__restrict__ off,
                                    const uint8_t *__restrict__ skip, int32_t *out) {
    const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= rows) return;
    const int64_t q = map ? map[r] : r;
    if (skip && skip[q]) return;
    const int64_t lo = off[q], len = min(off[q + 1] - lo, cap);  // (an overflowed row is re-run)
    for (int64_t i = lane_id(); i < len; i += 32) out[lo + i] = log[r * cap + i];
}

// CSR offsets of the visit logs from the iteration counts: off[0] = 0,
// off[i + 1] = off[i] + iters[i]; one CTA, chunk by chunk with a carry.
__global__ void __launch_bounds__(1024) scan_offsets_kernel(const int32_t *__restrict__ iters, int64_t n,
                                                            int64_t *__restrict__ off) {
    __shared__ long long s_w[32];
    __shared__ long long s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_carry = 0;
        off[0] = 0;
    }
    __syncthreads();
    for (int64_t base = 0; base < n; base += 1024) {
        const int64_t i = base + tid;
        long long v = i < n ? iters[i] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long u = __shfl_up_sync(0xFFFFFFFFu, v, o);
            if (lane >= o) v += u;
        }
        if (lane == 31) s_w[warp] = v;
        __syncthreads();
        if (warp == 0) {
            long long w = s_w[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long u = __shfl_up_sync(0xFFFFFFFFu, w, o);
                if (lane >= o) w += u;
            }
            s_w[lane] = w;
        }
        __syncthreads();
        const long long incl = v + (warp > 0 ? s_w[warp - 1] : 0) + s_carry;
        if (i < n) off[i + 1] = incl;
        __syncthreads();
        if (tid == 1023) s_carry = incl;
        __syncthreads();
    }
}

// exact_sq_dists (engine.py:48-51), row-paired, one thread per row.
__global__ void exact_dists_kernel(const void *points, int dtype, int dim,
                                   const float *__restrict__ queries, int64_t n, float *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = exact_sq_dist(points, dtype, dim, i, queries + i * dim);
}

}  // namespace bang

namespace bang {
// -------------------------------------------------------------------------
// Kernel 3 over a query-grouped pair list (north_star kernel 3; SURVEY.md
// 8(d) "a standalone ADC launch over all (query, neighbour) pairs"): one CTA
// per query builds the query's table in shared memory (kernel 1, pq.py:284-296
// op order), then every pair of that query gathers its PQ code row with
// 16-byte loads and sums the table entries sequentially in f32
// (engine.py:99-105).  keys[i] = f32bits << 32 | ids[i].  Code row i starts at
// codes + i * cstride.  Pairs of query q are
// ids[off[q], off[q+1]).  SUB/MV > 0: uniform subspaces of width SUB and
// m = 16*MV (vector path); 0: generic.
// -------------------------------------------------------------------------
#ifndef BANG_ADC_PAIRS_NT
#define BANG_ADC_PAIRS_NT 256
#endif
template <int SUB, int MV>
__global__ void __launch_bounds__(BANG_ADC_PAIRS_NT) adc_pairs_kernel(const float *__restrict__ centroids,
                                                        const int32_t *__restrict__ sub_off,
                                                        const int32_t *__restrict__ sub_size, int m,
                                                        int dim, const float *__restrict__ queries,
                                                        int64_t nq, const int64_t *__restrict__ off,
                                                        const uint32_t *__restrict__ ids,
                                                        const uint8_t *__restrict__ codes, int cstride,
                                                        uint64_t *__restrict__ keys) {
    extern __shared__ __align__(16) float s_tab[];  // m*256 table, then the query
    float *s_q = s_tab + (size_t)m * 256;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int64_t q = blockIdx.x; q < nq; q += gridDim.x) {
        for (int i = tid; i < dim; i += nt) s_q[i] = __ldg(queries + q * dim + i);
        __syncthreads();
        for (int idx = tid; idx < m * 256; idx += nt) {
            const int s = idx >> 8, c = idx & 255;
            float e;
            if constexpr (SUB == 4) {
                e = table_entry4(*reinterpret_cast<const float4 *>(s_q + s * 4),
                                 __ldg(reinterpret_cast<const float4 *>(centroids) + s * 256 + c));
            } else if constexpr (SUB == 2) {
                e = table_entry2(*reinterpret_cast<const float2 *>(s_q + s * 2),
                                 __ldg(reinterpret_cast<const float2 *>(centroids) + s * 256 + c));
            } else {
                const int o = __ldg(sub_off + s), sz = __ldg(sub_size + s);
                e = table_entry(s_q + o, centroids + (int64_t)o * 256 + c * sz, sz);
            }
            s_tab[idx] = e;
        }
        __syncthreads();
        const int64_t lo = off[q], hi = off[q + 1];
        if constexpr (MV > 0) {
            // Per warp, rounds of 32 pairs: the 32 code rows are copied into
            // the warp's smem stage by cp.async with MV consecutive lanes per
            // row (coalesced 16-byte pieces, no registers held), double
            // buffered so round r+1's rows are in flight while round r sums.
            constexpr int M = 16 * MV;
            const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
            uint8_t *stage = reinterpret_cast<uint8_t *>(s_q + ((dim + 3) & ~3)) + (size_t)warp * 2 * 32 * M;
            const int64_t nround = (hi - lo + 31) / 32;
            auto issue = [&](int64_t r, int buf) -> uint32_t {
                const int64_t base = lo + r * 32;
                const uint32_t my = base + lane < hi ? __ldg(ids + base + lane) : 0u;
#pragma unroll
                for (int v = 0; v < MV; ++v) {
                    const int ci = v * 32 + lane, row = ci / MV, part = ci - row * MV;
                    const uint32_t rid = __shfl_sync(kFull, my, row);
                    if (base + row < hi)
                        __pipeline_memcpy_async(stage + (size_t)buf * 32 * M + ci * 16,
                                                codes + (int64_t)rid * cstride + part * 16, 16);
                }
                __pipeline_commit();
                return my;
            };
            int64_t r = warp;
            uint32_t cur = r < nround ? issue(r, 0) : 0u;
            for (int k = 0; r < nround; ++k, r += nw) {
                const int64_t rn = r + nw;
                uint32_t nxt = 0u;
                if (rn < nround) {
                    nxt = issue(rn, (k + 1) & 1);
                    __pipeline_wait_prior(1);
                } else {
                    __pipeline_wait_prior(0);
                }
                __syncwarp();
                const int64_t i = lo + r * 32 + lane;
                if (i < hi) {
                    const uint4 *row = reinterpret_cast<const uint4 *>(stage + (size_t)(k & 1) * 32 * M + lane * M);
                    float a = 0.0f;
#pragma unroll
                    for (int v = 0; v < MV; ++v) a = adc_tab_stage16(a, s_tab, 16 * v, row[v]);
                    keys[i] = pack_key(a, cur);
                }
                __syncwarp();  // this buffer is refilled two rounds later
                cur = nxt;
            }
        } else {
            for (int64_t i = lo + tid; i < hi; i += nt) {
                const uint32_t node = __ldg(ids + i);
                keys[i] = pack_key(adc_table<0>(s_tab, m, codes + (int64_t)node * cstride), node);
            }
        }
        __syncthreads();
    }
}

}  // namespace bang
