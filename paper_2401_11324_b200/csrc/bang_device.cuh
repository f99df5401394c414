// bang_device.cuh -- device building blocks of the B200 BANG search path.
//
// Each function restates one piece of the reference's arithmetic (paths
// under /root/reference/pkg/src/bang/) so that every result is bit-exact:
//   f32 distance-table entries without FMA ....... pq.py:284-296
//   sequential f32 ADC sums over s = 0..m-1 ....... engine.py:99-105
//   FNV-1a-64 Bloom slots + test-and-set .......... bloom.py:26-42, 101-163
//   (f32 bits << 32 | id) keys and their order .... kernels.py:1-41
//   f64-accumulated exact distances -> f32 ....... engine.py:48-51
// They are shared by the fused persistent search kernel and by the
// stand-alone per-kernel entry points in bang_kernels.cuh.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace bang {

constexpr uint64_t kSentinel = 0xFFFFFFFFFFFFFFFFull;
constexpr uint64_t kFnvOffset = 0xCBF29CE484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001B3ull;
// h2 starts from FNV-1a of the prefix byte 0x5A (bloom.py:31-32)
constexpr uint64_t kFnvOffsetH2 = (kFnvOffset ^ 0x5Aull) * kFnvPrime;
constexpr unsigned kFull = 0xFFFFFFFFu;

enum VecDtype { kVecF32 = 0, kVecU8 = 1, kVecI8 = 2 };
// 0: CTA-shared codebook, entries recomputed per lookup; 1: HBM table built by
// kernel 1; 2: exact distances (exact_distance mode); 3: per-query table in
// the warp's shared memory, built at query start (the paper's layout).
enum AdcVariant { kAdcSmemCodebook = 0, kAdcGlobalTable = 1, kAdcExact = 2, kAdcSmemTable = 3 };

// kernels.py:25-29 -- non-negative f32 bit patterns are monotone, so the
// u64 order is the (dist, id) lexicographic order.
__host__ __device__ __forceinline__ uint64_t pack_key(float d, uint32_t id) {
#ifdef __CUDA_ARCH__
    return (static_cast<uint64_t>(__float_as_uint(d)) << 32) | id;
#else
    uint32_t b;
    __builtin_memcpy(&b, &d, 4);
    return (static_cast<uint64_t>(b) << 32) | id;
#endif
}
__device__ __forceinline__ float key_dist(uint64_t k) { return __uint_as_float((uint32_t)(k >> 32)); }
__device__ __forceinline__ uint32_t key_id(uint64_t k) { return (uint32_t)(k & 0xFFFFFFFFull); }

// bloom.py:26-34 -- FNV-1a-64 over the id's four little-endian bytes.
__host__ __device__ __forceinline__ uint64_t fnv1a(uint32_t id, uint64_t h) {
#pragma unroll
    for (int s = 0; s < 32; s += 8) h = (h ^ ((id >> s) & 0xFFu)) * kFnvPrime;
    return h;
}

// h mod z for a runtime z < 2^32 without the 64-bit division subroutine:
// magic = floor((2^64-1)/z) makes umulhi(h, magic) either floor(h/z) or one
// less (the truncation error is < 1), so one conditional subtract is exact.
struct BloomGeom {
    uint64_t z;
    uint64_t magic;
};
__device__ __forceinline__ uint32_t mod_z(uint64_t h, const BloomGeom &g) {
    uint64_t q = __umul64hi(h, g.magic);
    uint64_t r = h - q * g.z;
    if (r >= g.z) r -= g.z;
    return (uint32_t)r;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        uint64_t w = __shfl_xor_sync(kFull, v, o);
        v = w < v ? w : v;
    }
    return v;
}

// ---------------------------------------------------------------- Bloom
// One warp test-and-sets one row's probes (up to NPL*32 ids, probe i lives
// in lane i%32, register i/32) against one filter of u32 words.
// Semantics = sequential test-and-set in probe order (bloom.py:124-163):
//  1. every probe tests the PRE-state (two L2 loads issued together);
//  2. fresh probes set their bits with fetch-or atomics; a bit that another
//     fresh probe of this row set first shows up in the returned old word
//     while it was clear in the pre-state -- exactly the in-row slot
//     sharing that bloom.py:134-158 detects;
//  3. on such a collision (rare: ~0.3% of rows at z = 399,887) the touched
//     words are restored to the pre-state and lane 0 replays the row in
//     order (bloom.py:110-122) -- bit-exact, unlike the paper's tolerated
//     race.
// Phase 2 is split (bloom_issue / bloom_resolve) so the atomics' round trip
// overlaps the ADC of the fresh neighbours.
//
// Optional per-warp summary (s_sum != nullptr; the fused search kernel):
// one smem bit per filter word, set when the word is first written by the
// current query.  A word whose summary bit is clear holds garbage from an
// earlier query and is read as 0 without touching memory, so the 50 KB
// filter never needs clearing and only words this query wrote are ever
// read (most probes then cost no load at all).  The filter state it
// represents is identical: bit p is set <=> summary(p>>5) && word(p>>5) has p.
// Filters are read through L2 (ld.global.cg): they are written by atomics
// performed at L2 during the same kernel.
template <int NPL>
struct BloomRow {
    uint32_t p1[NPL], p2[NPL], w1[NPL], w2[NPL], o1[NPL], o2[NPL];
    bool i1[NPL], i2[NPL];  // word was initialised before this row (summary)
    bool fresh[NPL];
};

__device__ __forceinline__ bool sum_get(const uint32_t *s_sum, uint32_t w) {
    return (s_sum[w >> 5] >> (w & 31)) & 1u;
}
__device__ __forceinline__ void sum_set(uint32_t *s_sum, uint32_t w) {
    atomicOr(s_sum + (w >> 5), 1u << (w & 31));
}

template <int NPL>
__device__ __forceinline__ void bloom_issue(uint32_t *__restrict__ bits, uint32_t *s_sum,
                                            const BloomGeom &g, const uint32_t (&ids)[NPL],
                                            int cnt, BloomRow<NPL> &b) {
    const int lane = (int)lane_id();
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
        b.fresh[k] = false;
        b.p1[k] = b.p2[k] = b.w1[k] = b.w2[k] = b.o1[k] = b.o2[k] = 0;
        b.i1[k] = b.i2[k] = true;
        if (lane + 32 * k < cnt) {
            b.p1[k] = mod_z(fnv1a(ids[k], kFnvOffset), g);
            b.p2[k] = mod_z(fnv1a(ids[k], kFnvOffsetH2), g);
            if (s_sum) {
                b.i1[k] = sum_get(s_sum, b.p1[k] >> 5);
                b.i2[k] = sum_get(s_sum, b.p2[k] >> 5);
            }
            if (b.i1[k]) b.w1[k] = __ldcg(bits + (b.p1[k] >> 5));
            if (b.i2[k]) b.w2[k] = __ldcg(bits + (b.p2[k] >> 5));
        }
    }
#pragma unroll
    for (int k = 0; k < NPL; ++k)
        if (lane + 32 * k < cnt)
            b.fresh[k] = !(((b.w1[k] >> (b.p1[k] & 31)) & 1u) && ((b.w2[k] >> (b.p2[k] & 31)) & 1u));
    __syncwarp();  // every pre-state load has landed before any write below
    if (s_sum) {
        // words first written by this query: zero them and mark the summary
        bool any = false;
#pragma unroll
        for (int k = 0; k < NPL; ++k) {
            if (b.fresh[k] && !b.i1[k]) {
                __stcg(bits + (b.p1[k] >> 5), 0u);
                sum_set(s_sum, b.p1[k] >> 5);
                any = true;
            }
            if (b.fresh[k] && !b.i2[k]) {
                __stcg(bits + (b.p2[k] >> 5), 0u);
                sum_set(s_sum, b.p2[k] >> 5);
                any = true;
            }
        }
        if (__any_sync(kFull, any)) {
            __threadfence_block();
            __syncwarp();  // the zeroing stores are ordered before the atomics
        }
    }
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
        if (b.fresh[k]) {
            b.o1[k] = atomicOr(bits + (b.p1[k] >> 5), 1u << (b.p1[k] & 31));
            if (b.p2[k] != b.p1[k]) b.o2[k] = atomicOr(bits + (b.p2[k] >> 5), 1u << (b.p2[k] & 31));
        }
    }
}

// Checks the atomics' old words; on an in-row collision restores the
// pre-state and replays the row sequentially.  Returns true (warp-uniform)
// when the fresh set was recomputed.
template <int NPL>
__device__ __forceinline__ bool bloom_resolve(uint32_t *__restrict__ bits, uint32_t *s_sum,
                                              const BloomGeom &g, const uint32_t (&ids)[NPL],
                                              int cnt, BloomRow<NPL> &b) {
    const int lane = (int)lane_id();
    bool coll = false;
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
        if (b.fresh[k]) {
            const uint32_t b1 = 1u << (b.p1[k] & 31);
            coll |= (b.o1[k] & b1) && !(b.w1[k] & b1);
            if (b.p2[k] != b.p1[k]) {
                const uint32_t b2 = 1u << (b.p2[k] & 31);
                coll |= (b.o2[k] & b2) && !(b.w2[k] & b2);
            }
        }
    }
    if (!__any_sync(kFull, coll)) {
        __syncwarp();
        return false;
    }
    // restore the pre-state of every word a fresh probe touched
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
        if (b.fresh[k]) {
            if (b.i1[k]) __stcg(bits + (b.p1[k] >> 5), b.w1[k]);
            if (b.i2[k]) __stcg(bits + (b.p2[k] >> 5), b.w2[k]);
        }
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
        if (b.fresh[k] && s_sum) {
            if (!b.i1[k]) atomicAnd(s_sum + ((b.p1[k] >> 5) >> 5), ~(1u << ((b.p1[k] >> 5) & 31)));
            if (!b.i2[k]) atomicAnd(s_sum + ((b.p2[k] >> 5) >> 5), ~(1u << ((b.p2[k] >> 5) & 31)));
        }
    }
    __threadfence_block();
    __syncwarp();
    // sequential replay in appearance order (lane 0)
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
        uint32_t mask = 0;
        const int n = min(32, cnt - 32 * k);
        for (int j = 0; j < n; ++j) {
            const uint32_t id = __shfl_sync(kFull, ids[k], j);
            if (lane == 0) {
                const uint32_t q[2] = {mod_z(fnv1a(id, kFnvOffset), g), mod_z(fnv1a(id, kFnvOffsetH2), g)};
                bool hit = true;
                for (int h = 0; h < 2; ++h) {
                    const uint32_t w = q[h] >> 5;
                    const bool init = !s_sum || sum_get(s_sum, w);
                    hit = hit && init && ((__ldcg(bits + w) >> (q[h] & 31)) & 1u);
                }
                if (!hit) {
                    for (int h = 0; h < 2; ++h) {
                        const uint32_t w = q[h] >> 5;
                        if (s_sum && !sum_get(s_sum, w)) {
                            __stcg(bits + w, 1u << (q[h] & 31));
                            s_sum[w >> 5] |= 1u << (w & 31);
                        } else {
                            atomicOr(bits + w, 1u << (q[h] & 31));
                        }
                    }
                    mask |= 1u << j;
                }
            }
        }
        mask = __shfl_sync(kFull, mask, 0);
        b.fresh[k] = (mask >> lane) & 1u;
    }
    __threadfence_block();
    __syncwarp();
    return true;
}

// In-row slot sharing, exact replay by one warp from the pre-state bits the
// row's probes already loaded -- no L2 round trips (bloom.py:110-122,
// 134-158).  Inputs (shared memory, probe j = 0..deg-1):
//   rec[j] = (p1, p2) slots; fl2[2j + h] per half h: bit 1 presumed fresh
//   (pre-state test), bit 2 pre-state bit of slot h, bit 3 this half's
//   fetch-or found its bit set by another probe of the row.
// Every presumed-fresh probe already set its bits with fetch-or.  Only
// presumed-fresh probes that share a slot can change the sequential outcome
// (a shared slot always shows up as a collision on one of its fetch-ors), so
// those "involved" probes are replayed in adjacency order; dropped probes'
// bits that neither the pre-state nor a truly fresh probe holds are cleared.
// Output tf[j] = truly fresh (j < RPAD).
template <int NPL>
__device__ __forceinline__ int replay_row_warp(const uint2 *rec, const uint8_t *fl2, int deg,
                                               uint32_t *bits, uint8_t *tf_out) {
    const int lane = (int)lane_id();
    uint32_t a[NPL], b[NPL];
    bool pf[NPL], pre1[NPL], pre2[NPL], inv[NPL], tf[NPL], dr[NPL];
#pragma unroll
    for (int r = 0; r < NPL; ++r) {
        const int jj = lane + 32 * r;
        const bool in = jj < deg;
        const uint2 v = in ? rec[jj] : make_uint2(0u, 0u);
        const uint8_t f0 = in ? fl2[2 * jj] : 0, f1 = in ? fl2[2 * jj + 1] : 0;
        a[r] = v.x;
        b[r] = v.y;
        pf[r] = (f0 & 2) != 0;
        pre1[r] = (f0 & 4) != 0;
        pre2[r] = (f1 & 4) != 0;
        inv[r] = pf[r] && ((f0 | f1) & 8);
        tf[r] = dr[r] = false;
    }
    // partners: presumed-fresh probes sharing a slot with a colliding one
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
    auto in_set = [&](uint32_t pos) {  // slot set by an earlier truly fresh involved probe
        bool hit = false;
#pragma unroll
        for (int r = 0; r < NPL; ++r) hit = hit || (tf[r] && (a[r] == pos || b[r] == pos));
        return __any_sync(kFull, hit);
    };
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
    int ndrop = 0;
#pragma unroll
    for (int r = 0; r < NPL; ++r) {
        unsigned dm = __ballot_sync(kFull, dr[r]);
        ndrop += __popc(dm);
        while (dm) {
            const int src = __ffs(dm) - 1;
            dm &= dm - 1;
            const uint32_t pa = __shfl_sync(kFull, a[r], src), pb = __shfl_sync(kFull, b[r], src);
            const bool q1 = __shfl_sync(kFull, (int)pre1[r], src), q2 = __shfl_sync(kFull, (int)pre2[r], src);
            const bool keep_a = q1 || in_set(pa);
            const bool keep_b = pb == pa || q2 || in_set(pb);
            if (lane == 0) {
                if (!keep_a) atomicAnd(bits + (pa >> 5), ~(1u << (pa & 31)));
                if (!keep_b) atomicAnd(bits + (pb >> 5), ~(1u << (pb & 31)));
            }
        }
    }
#pragma unroll
    for (int r = 0; r < NPL; ++r) tf_out[lane + 32 * r] = (uint8_t)(pf[r] && !dr[r]);
    return ndrop;
}

// Both phases back to back (the stand-alone bank kernel).
template <int NPL>
__device__ __forceinline__ void bloom_test_and_set(uint32_t *__restrict__ bits, uint32_t *s_sum,
                                                   const BloomGeom &g,
                                                   const uint32_t (&ids)[NPL], int cnt,
                                                   bool (&fresh)[NPL]) {
    BloomRow<NPL> b;
    bloom_issue<NPL>(bits, s_sum, g, ids, cnt, b);
    bloom_resolve<NPL>(bits, s_sum, g, ids, cnt, b);
#pragma unroll
    for (int k = 0; k < NPL; ++k) fresh[k] = b.fresh[k];
}

// ------------------------------------------------------- distance table
// pq.py:290-294: diff = q - c; diff *= diff; acc = diff[0]; acc += diff[j].
// Intrinsics keep every op separately rounded (no FFMA contraction).
__device__ __forceinline__ float table_entry(const float *__restrict__ q,
                                             const float *__restrict__ c, int size) {
    float d = __fsub_rn(q[0], c[0]);
    float acc = __fmul_rn(d, d);
    for (int j = 1; j < size; ++j) {
        d = __fsub_rn(q[j], c[j]);
        acc = __fadd_rn(acc, __fmul_rn(d, d));
    }
    return acc;
}
__device__ __forceinline__ float table_entry2(float2 q, float2 c) {
    float d0 = __fsub_rn(q.x, c.x), d1 = __fsub_rn(q.y, c.y);
    return __fadd_rn(__fmul_rn(d0, d0), __fmul_rn(d1, d1));
}
__device__ __forceinline__ float table_entry4(float4 q, float4 c) {
    float d0 = __fsub_rn(q.x, c.x), d1 = __fsub_rn(q.y, c.y);
    float d2 = __fsub_rn(q.z, c.z), d3 = __fsub_rn(q.w, c.w);
    float acc = __fadd_rn(__fmul_rn(d0, d0), __fmul_rn(d1, d1));
    acc = __fadd_rn(acc, __fmul_rn(d2, d2));
    return __fadd_rn(acc, __fmul_rn(d3, d3));
}

// Per-query table in shared memory (variant D): entries of pq.py:290-294 for
// all (s, c), written by the warp's lanes; centroids read from global/L2.
template <int SUB>
__device__ __forceinline__ void build_table_warp(float *s_tab, const float *__restrict__ s_q,
                                                 const float *__restrict__ centroids,
                                                 const int32_t *__restrict__ sub_off,
                                                 const int32_t *__restrict__ sub_size, int m) {
    for (int idx = (int)lane_id(); idx < m * 256; idx += 32) {
        const int s = idx >> 8, c = idx & 255;
        float e;
        if constexpr (SUB == 4) {
            e = table_entry4(*reinterpret_cast<const float4 *>(s_q + s * 4),
                             __ldg(reinterpret_cast<const float4 *>(centroids) + s * 256 + c));
        } else if constexpr (SUB == 2) {
            e = table_entry2(*reinterpret_cast<const float2 *>(s_q + s * 2),
                             __ldg(reinterpret_cast<const float2 *>(centroids) + s * 256 + c));
        } else {
            const int off = __ldg(sub_off + s), sz = __ldg(sub_size + s);
            const float *src = centroids + (int64_t)off * 256 + c * sz;
            float dd = __fsub_rn(s_q[off], __ldg(src));
            float acc = __fmul_rn(dd, dd);
            for (int j = 1; j < sz; ++j) {
                dd = __fsub_rn(s_q[off + j], __ldg(src + j));
                acc = __fadd_rn(acc, __fmul_rn(dd, dd));
            }
            e = acc;
        }
        s_tab[idx] = e;
    }
}

// ------------------------------------------------------------------ ADC
// engine.py:99-105: acc = 0f; acc += T[s][code[s]] for s = 0..m-1 (f32).
// Variant A (smem codebook): T[s][c] is recomputed from the CTA-resident
// codebook and the warp's query in exactly pq.py's op order, so it equals
// the table entry bit-for-bit (verified by the parity tests).
// SUB > 0: uniform subspace width; MV > 0: m = 16*MV, code rows read as MV
// 16-byte vectors (north_star's vectorised code gather).
template <int SUB, int MV>
__device__ __forceinline__ float adc_codebook(const float *__restrict__ s_cb,
                                              const float *__restrict__ s_q,
                                              const int *__restrict__ s_off,
                                              const int *__restrict__ s_sz, int m,
                                              const uint8_t *__restrict__ code_row) {
    float acc = 0.0f;
    if constexpr (SUB > 0 && MV > 0) {
        uint4 cv[MV];
#pragma unroll
        for (int v = 0; v < MV; ++v) cv[v] = __ldg(reinterpret_cast<const uint4 *>(code_row) + v);
#pragma unroll
        for (int v = 0; v < MV; ++v) {
            const uint32_t w[4] = {cv[v].x, cv[v].y, cv[v].z, cv[v].w};
#pragma unroll
            for (int b = 0; b < 16; ++b) {
                const int s = v * 16 + b;
                const uint32_t c = (w[b >> 2] >> ((b & 3) * 8)) & 0xFFu;
                float e;
                if constexpr (SUB == 4) {
                    e = table_entry4(*reinterpret_cast<const float4 *>(s_q + s * 4),
                                     *reinterpret_cast<const float4 *>(s_cb + (s * 256 + c) * 4));
                } else if constexpr (SUB == 2) {
                    e = table_entry2(*reinterpret_cast<const float2 *>(s_q + s * 2),
                                     *reinterpret_cast<const float2 *>(s_cb + (s * 256 + c) * 2));
                } else {
                    e = table_entry(s_q + s * SUB, s_cb + (s * 256 + c) * SUB, SUB);
                }
                acc = __fadd_rn(acc, e);
            }
        }
    } else {
        for (int s = 0; s < m; ++s) {
            const int c = __ldg(code_row + s);
            const int off = s_off[s], sz = s_sz[s];
            acc = __fadd_rn(acc, table_entry(s_q + off, s_cb + off * 256 + c * sz, sz));
        }
    }
    return acc;
}

// Variants B/D (table from kernel 1 in HBM, or the warp's smem table): the
// reference's literal data flow.  Plain loads: trow may point to either.
template <int MV>
__device__ __forceinline__ float adc_table(const float *trow, int m,
                                           const uint8_t *__restrict__ code_row) {
    float acc = 0.0f;
    if constexpr (MV > 0) {
        uint4 cv[MV];
#pragma unroll
        for (int v = 0; v < MV; ++v) cv[v] = __ldg(reinterpret_cast<const uint4 *>(code_row) + v);
#pragma unroll
        for (int v = 0; v < MV; ++v) {
            const uint32_t w[4] = {cv[v].x, cv[v].y, cv[v].z, cv[v].w};
#pragma unroll
            for (int b = 0; b < 16; ++b) {
                const int s = v * 16 + b;
                const uint32_t c = (w[b >> 2] >> ((b & 3) * 8)) & 0xFFu;
                acc = __fadd_rn(acc, trow[s * 256 + c]);
            }
        }
    } else {
        for (int s = 0; s < m; ++s) acc = __fadd_rn(acc, trow[s * 256 + __ldg(code_row + s)]);
    }
    return acc;
}

// ------------------------------------------------------ exact distances
// Plain loads: the vectors may live in pinned, mapped host memory.
// engine.py:48-51: widen to f32 (validation.py:38-43), f64 difference,
// f64 sum of squares in dimension order, round to f32.  (numpy's einsum
// sums in a SIMD order; the rounded f32 agrees -- SURVEY.md 8(c).)
__device__ __forceinline__ float exact_sq_dist(const void *__restrict__ vectors, int dtype,
                                               int dim, int64_t row,
                                               const float *__restrict__ q) {
    double acc = 0.0;
    if (dtype == kVecF32) {
        const float *x = reinterpret_cast<const float *>(vectors) + row * (int64_t)dim;
        if ((dim & 3) == 0) {
            for (int j = 0; j < dim; j += 4) {
                const float4 v = *reinterpret_cast<const float4 *>(x + j);
                const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const double d = __dsub_rn((double)xs[u], (double)q[j + u]);
                    acc = __dadd_rn(acc, __dmul_rn(d, d));
                }
            }
        } else {
            for (int j = 0; j < dim; ++j) {
                const double d = __dsub_rn((double)x[j], (double)q[j]);
                acc = __dadd_rn(acc, __dmul_rn(d, d));
            }
        }
    } else {
        const uint8_t *x = reinterpret_cast<const uint8_t *>(vectors) + row * (int64_t)dim;
        const bool sgn = dtype == kVecI8;
        if ((dim & 3) == 0) {
            for (int j = 0; j < dim; j += 4) {
                const uint32_t v = *reinterpret_cast<const uint32_t *>(x + j);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t b = (v >> (8 * u)) & 0xFFu;
                    const float xf = sgn ? (float)(int8_t)b : (float)b;
                    const double d = __dsub_rn((double)xf, (double)q[j + u]);
                    acc = __dadd_rn(acc, __dmul_rn(d, d));
                }
            }
        } else {
            for (int j = 0; j < dim; ++j) {
                const uint32_t b = x[j];
                const float xf = sgn ? (float)(int8_t)b : (float)b;
                const double d = __dsub_rn((double)xf, (double)q[j]);
                acc = __dadd_rn(acc, __dmul_rn(d, d));
            }
        }
    }
    return __double2float_rn(acc);
}

// ------------------------------------------------------- sorted arrays
// number of entries of sorted a[0, n) strictly below x.  Binary lifting:
// the trip count depends on n only, so lanes searching different keys of
// the same array never diverge.
__device__ __forceinline__ int lower_bound_u64(const uint64_t *a, int n, uint64_t x) {
    int lo = 0;
    for (int step = n > 0 ? 1 << (31 - __clz(n)) : 0; step > 0; step >>= 1)
        if (lo + step <= n && a[lo + step - 1] < x) lo += step;
    return lo;
}
// number of entries of sorted a[0, n) at or below x
__device__ __forceinline__ int upper_bound_u64(const uint64_t *a, int n, uint64_t x) {
    int lo = 0;
    for (int step = n > 0 ? 1 << (31 - __clz(n)) : 0; step > 0; step >>= 1)
        if (lo + step <= n && a[lo + step - 1] <= x) lo += step;
    return lo;
}

// first index i in [from, cnt) with vis[i] == 0 (cnt if none); warp-uniform
__device__ __forceinline__ int first_unvisited(const uint8_t *s_vis, int from, int cnt) {
    const int lane = (int)lane_id();
    for (int b = from; b < cnt; b += 32) {
        const int i = b + lane;
        const unsigned m = __ballot_sync(kFull, i < cnt && !s_vis[i]);
        if (m) return b + __ffs(m) - 1;
    }
    return cnt;
}

// ------------------------------------------------ worklist sort + merge
// kernels.py:44-109 / engine.py:210-215 for one warp-owned worklist in smem.
// Keys in wl u new are unique (the Bloom filter has no false negatives), so
// any correct sort/merge is bit-identical to the reference's rank merge with
// its a-first tie rule.
//
// Only "survivors" reach the merge: when the worklist is full (cnt == t) a
// new key >= wl[t-1] would land at rank >= t and be truncated by
// merged[:, :t] (engine.py:213), so it is dropped before sorting.  The eager
// winner is unaffected: a dropped key can only be the minimum when every
// kept entry is visited, i.e. when the query converges this iteration.

// s_sk[rank] = s_nk[j]: rank = #keys below it (n <= 128, broadcast reads)
__device__ __forceinline__ void sort_keys(const uint64_t *s_nk, int n, uint64_t *s_sk) {
    const int lane = (int)lane_id();
    for (int j = lane; j < n; j += 32) {
        const uint64_t k = s_nk[j];
        int r = 0;
        for (int i = 0; i < n; ++i) r += s_nk[i] < k;
        s_sk[r] = k;
    }
    __syncwarp();
}

// Merge sorted survivors s_sk[0, n) into s_wl[0, cnt) (+ visited flags) and
// truncate to t: each element's final rank = own rank + rank in the other
// list (the paper's Merge_LSet).  Entries below the
// first insertion point do not move; the rest are moved in place chunk by
// chunk from the top so no unread entry is overwritten.  n <= 128.
__device__ __forceinline__ int merge_sorted(uint64_t *s_wl, uint8_t *s_vis, int cnt, int t,
                                            const uint64_t *s_sk, int n, int *first_out) {
    const int lane = (int)lane_id();
    if (n == 0) {
        *first_out = cnt;
        return cnt;
    }
    const int first = lower_bound_u64(s_wl, cnt, s_sk[0]);
    *first_out = first;
    int pos[4];
    uint64_t kv[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int j = lane + 32 * c;
        pos[c] = t;
        kv[c] = 0;
        if (j < n) {
            kv[c] = s_sk[j];
            pos[c] = j + first + lower_bound_u64(s_wl + first, cnt - first, kv[c]);
        }
    }
    __syncwarp();
    if (first < cnt) {
        for (int ch = (cnt - 1) >> 5; ch >= (first >> 5); --ch) {
            const int i = ch * 32 + lane;
            uint64_t v = 0;
            uint8_t vv = 0;
            int dst = t;
            if (i >= first && i < cnt) {
                v = s_wl[i];
                vv = s_vis[i];
                dst = i + lower_bound_u64(s_sk, n, v);
            }
            __syncwarp();
            if (dst < t) {
                s_wl[dst] = v;
                s_vis[dst] = vv;
            }
            __syncwarp();
        }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        if (pos[c] < t) {
            s_wl[pos[c]] = kv[c];
            s_vis[pos[c]] = 0;
        }
    }
    __syncwarp();
    return min(t, cnt + n);
}

// ------------------------------------------------------- staged ADC ranges
// acc += T[s][code_s] for s in [s0, s0 + 8) -- the same sequential f32 sum
// as adc_codebook/adc_table, split into 8-subspace stages so that a
// candidate whose partial sum already exceeds the worklist's last distance
// can be dropped (f32 addition of non-negative terms is monotone, so
// partial > thr implies final > thr: the survivor set is exact).
template <int SUB>
__device__ __forceinline__ float adc_cb_stage(float acc, const float *__restrict__ s_cb,
                                              const float *__restrict__ s_q,
                                              const int *__restrict__ s_off,
                                              const int *__restrict__ s_sz, int s0, int ns,
                                              uint64_t c8) {
    if constexpr (SUB > 0) {
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int s = s0 + b;
            const uint32_t c = (uint32_t)(c8 >> (8 * b)) & 0xFFu;
            float e;
            if constexpr (SUB == 4) {
                e = table_entry4(*reinterpret_cast<const float4 *>(s_q + s * 4),
                                 *reinterpret_cast<const float4 *>(s_cb + (s * 256 + c) * 4));
            } else if constexpr (SUB == 2) {
                e = table_entry2(*reinterpret_cast<const float2 *>(s_q + s * 2),
                                 *reinterpret_cast<const float2 *>(s_cb + (s * 256 + c) * 2));
            } else {
                e = table_entry(s_q + s * SUB, s_cb + (s * 256 + c) * SUB, SUB);
            }
            acc = __fadd_rn(acc, e);
        }
    } else {
        for (int b = 0; b < ns; ++b) {
            const int s = s0 + b;
            const int c = (int)((c8 >> (8 * b)) & 0xFFu);
            const int off = s_off[s], sz = s_sz[s];
            acc = __fadd_rn(acc, table_entry(s_q + off, s_cb + off * 256 + c * sz, sz));
        }
    }
    return acc;
}

__device__ __forceinline__ float adc_tab_stage(float acc, const float *trow, int s0,
                                               int ns, uint64_t c8) {
    for (int b = 0; b < ns; ++b)
        acc = __fadd_rn(acc, trow[(s0 + b) * 256 + (int)((c8 >> (8 * b)) & 0xFFu)]);
    return acc;
}

// eight code bytes of a row starting at subspace s0 (fewer at the tail)
template <bool ALIGNED8>
__device__ __forceinline__ uint64_t load_code8(const uint8_t *__restrict__ row, int s0, int ns) {
    if constexpr (ALIGNED8) {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(row + s0));
        return (uint64_t)v.x | ((uint64_t)v.y << 32);
    } else {
        uint64_t c8 = 0;
        for (int b = 0; b < ns; ++b) c8 |= (uint64_t)__ldg(row + s0 + b) << (8 * b);
        return c8;
    }
}

}  // namespace bang

namespace bang {
// 16-subspace stages for rows of m = 16*MV codes read as uint4 vectors.
template <int SUB>
__device__ __forceinline__ float adc_cb_stage16(float acc, const float *__restrict__ s_cb,
                                                const float *__restrict__ s_q, int s0, uint4 cv) {
    const uint32_t w[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
    for (int b = 0; b < 16; ++b) {
        const int s = s0 + b;
        const uint32_t c = (w[b >> 2] >> ((b & 3) * 8)) & 0xFFu;
        float e;
        if constexpr (SUB == 4) {
            e = table_entry4(*reinterpret_cast<const float4 *>(s_q + s * 4),
                             *reinterpret_cast<const float4 *>(s_cb + (s * 256 + c) * 4));
        } else if constexpr (SUB == 2) {
            e = table_entry2(*reinterpret_cast<const float2 *>(s_q + s * 2),
                             *reinterpret_cast<const float2 *>(s_cb + (s * 256 + c) * 2));
        } else {
            e = table_entry(s_q + s * SUB, s_cb + (s * 256 + c) * SUB, SUB);
        }
        acc = __fadd_rn(acc, e);
    }
    return acc;
}

__device__ __forceinline__ float adc_tab_stage16(float acc, const float *trow, int s0,
                                                 uint4 cv) {
    const uint32_t w[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
    for (int b = 0; b < 16; ++b)
        acc = __fadd_rn(acc, trow[(s0 + b) * 256 + ((w[b >> 2] >> ((b & 3) * 8)) & 0xFFu)]);
    return acc;
}
}  // namespace bang
