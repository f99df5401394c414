// bang_search_split.cuh -- one CTA per query with the iteration split into two
// concurrent roles (the paper's one-hop-ahead pipeline, PAPER.md:922-938,
// carried through the whole memory phase of a hop):
//
//   row warps  (warps 0-1, one thread per neighbour slot): for the node just
//              chosen, load its adjacency row, hash every id into its two
//              Bloom slots (bloom.py:26-42), read the pre-state bits, perform
//              the row's sets (fetch-or), gather the code rows straight into
//              registers and sum their ADC distances from the smem table
//              (engine.py:99-105); exact in-row slot sharing is replayed
//              (bloom.py:110-163).  Output: the row's keys in shared memory
//              and their minimum.
//   list warps (warps 2-3): meanwhile merge the PREVIOUS row's survivors into
//              the worklist (kernels.py:44-109, engine.py:210-215), mark and
//              log the node being expanded (engine.py:167-178) and find the
//              next unvisited head.
//
// They meet once per hop at one CTA barrier.  There the eager winner of the
// next hop is min(row minimum, head) (engine.py:201-205) and convergence is
// "no unvisited head and no row key below the truncation threshold"
// (engine.py:217): the post-merge worklist is all-visited exactly then.  So
// the critical path of a hop is the row chain alone (row -> {Bloom words,
// code rows} -> ADC); sort and merge run off it.
//
// Semantics are SURVEY.md 8(a0) bit for bit (same as search_cta_kernel).
#pragma once

#include "bang_search_cta.cuh"

// table entries (centroid loads) in flight per prologue thread (8, 16 and
// 24 measured equal, profiles/r02/ab_h/)
#ifndef BANG_TAB_UNROLL
#define BANG_TAB_UNROLL 8
#endif

namespace bang {

constexpr int kTabUnroll = BANG_TAB_UNROLL;

// L2 residency of the per-query Bloom filters.  A query's ~17 K fetch-ors hit
// random words of its 50 KB filter over ~0.5 ms while ~0.6 GB of code rows,
// adjacency rows and vectors stream through the 126 MB L2; ncu counted half
// of the fetch-ors as L2 misses (109 M of 220 M atomic sectors, under ncu's
// cache control).  The fetch-ors carry an evict_last policy (+0.5%, so the
// misses are mostly an artefact of the capture); hinted loads/stores of the
// filter measured neutral and a hinted cp.async of the code rows faulted
// (illegal instruction) on the B200, so those stay plain
// (profiles/r02/ab_g/, ab_h/).
__device__ __forceinline__ uint64_t l2_keep() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint32_t bloom_or(uint32_t *a, uint32_t v) {
    uint32_t o;
    asm volatile("atom.global.or.L2::cache_hint.b32 %0, [%1], %2, %3;" : "=r"(o) : "l"(a), "r"(v), "l"(l2_keep()) : "memory");
    return o;
}
__device__ __forceinline__ uint32_t bloom_ld(const uint32_t *a) { return __ldcg(a); }
__device__ __forceinline__ void bloom_st(uint32_t *a, uint32_t v) { __stcg(a, v); }
__device__ __forceinline__ void bloom_st4(uint4 *a, uint4 v) { __stcg(a, v); }
__device__ __forceinline__ void code_copy16(void *dst, const void *src) { __pipeline_memcpy_async(dst, src, 16); }

struct SplitMisc {
    unsigned long long rmin[2][2];  // [parity][row warp]: min key of the row's fresh neighbours
    unsigned long long head[2];  // [parity]: first unvisited worklist key (SENTINEL if none)
    unsigned long long thr[2];   // [parity]: wl[t-1] when the worklist is full, else SENTINEL
    unsigned long long okey;     // list warps: next unvisited old entry after the winner
    int rfresh[2][2];            // [parity][row warp]: fresh neighbours of the row
    int rdeg[2];                 // [parity]: degree of the row
    int hpos[2];                 // [parity]: position of the head
    int cnt[2];                  // [parity]: worklist entries
    int wsurv[2];                // list warps: survivors per list warp
    int opos;                    // list warps: old position of okey (cnt if none)
    int coll;                    // row warps: in-row slot sharing seen
    long long qi;
    uint32_t hid;                // HEADROW: node whose row ids are staged in s_hrow (~0u: none)
    int32_t hdeg;                // HEADROW: its deg_share word
    unsigned long long ph[8];  // phase profiler
};
static_assert(sizeof(SplitMisc) <= 256, "SplitMisc must fit its 256-byte smem slot");

// named barrier over a subset of the CTA's warps
__device__ __forceinline__ void split_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// adjacency row + degree of node v towards L2 (a candidate for the next
// winner, PAPER.md:922-938 one hop ahead)
__device__ __forceinline__ void prefetch_row_l2(const SearchParams &p, uint32_t v) {
    const int32_t *row = p.adj + (int64_t)v * p.adj_stride;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(row) : "memory");
    if (((uintptr_t)row & 127u) + 4u * (uint32_t)p.R > 128u)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(row + p.R - 1) : "memory");
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p.deg_share ? p.deg_share + v : p.deg + v) : "memory");
}
// clock64 read that waits for v (a value loaded earlier): the profiler's
// stamps must depend on the use they time
__device__ __forceinline__ long long clock_after(int v) {
    long long c;
    asm volatile("{\n\t.reg .u32 t;\n\tmov.u32 t, %1;\n\tmov.u64 %0, %%clock64;\n\t}" : "=l"(c) : "r"(v) : "memory");
    return c;
}

// 16 bytes of a code row; read-only for the kernel's lifetime, used once
__device__ __forceinline__ uint4 ldg_code16(const uint8_t *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t u4_word(const uint4 &v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// warp_topk_write over keys in shared memory: k rounds of "smallest key
// above the last one" (keys are unique), ids -1 / dists +inf padded
__device__ __forceinline__ void warp_topk_write_smem(const uint64_t *keys, int L, int k, int32_t *out_ids,
                                                     float *out_dists) {
    const int lane = (int)lane_id();
    uint64_t last = 0;
    for (int j = 0; j < k; ++j) {
        uint64_t local = kSentinel;
        if (j < L)
            for (int i = lane; i < L; i += 32) {
                const uint64_t v = keys[i];
                if ((j == 0 || v > last) && v < local) local = v;
            }
        const uint64_t sel = warp_min_u64(local);
        if (lane == 0) {
            out_ids[j] = sel != kSentinel ? (int32_t)key_id(sel) : -1;
            out_dists[j] = sel != kSentinel ? key_dist(sel) : __int_as_float(0x7f800000);
        }
        last = sel;
    }
}

// Rare path of split_row (~2% of rows at z = 399,887), kept out of line so
// the hop loop's code stays compact: exact sequential replay of the involved
// probes by row warp 0 from the pre-state bits; the records go where the
// (consumed) code rows were staged.  All 64 row threads call it; the probe
// state travels by value (registers) and the truly fresh flags come back as
// a bit mask (bit r: slot rt + 64 r).
template <int PL>
struct RowProbes {
    uint32_t p1[PL], p2[PL];
    uint32_t pf, b1, b2, sh1, sh2;  // bit r: slot rt + 64 r
};
template <int PL>
__device__ __noinline__ uint32_t split_replay(int rt, int deg, const RowProbes<PL> pr, uint8_t *s_stage,
                                              uint32_t *bits, uint8_t *s_tf) {
    constexpr int RPAD = 64 * PL;
    uint2 *s_rec = reinterpret_cast<uint2 *>(s_stage);
    uint8_t *s_fl2 = s_stage + 8 * RPAD;
    split_bar(3, 64);  // every row thread has read its staged rows
#pragma unroll
    for (int r = 0; r < PL; ++r) {
        const int jj = rt + 64 * r;
        const uint32_t m = 1u << r;
        s_rec[jj] = make_uint2(pr.p1[r], pr.p2[r]);
        s_fl2[2 * jj] = (uint8_t)((pr.pf & m ? 2 : 0) | (pr.b1 & m ? 4 : 0) | (pr.sh1 & m ? 8 : 0));
        s_fl2[2 * jj + 1] = (uint8_t)((pr.b2 & m ? 4 : 0) | (pr.sh2 & m ? 8 : 0));
    }
    split_bar(3, 64);
    if ((rt >> 5) == 0) replay_row_warp<RPAD / 32>(s_rec, s_fl2, deg, bits, s_tf);
    split_bar(3, 64);
    uint32_t fresh = 0;
#pragma unroll
    for (int r = 0; r < PL; ++r)
        if (rt + 64 * r < deg && s_tf[rt + 64 * r]) fresh |= 1u << r;
    return fresh;
}

// ADC of this thread's staged code rows whose flag is set: acc = ((0 +
// T[0][c0]) + T[1][c1]) + ... in f32 (engine.py:99-105); the lookups of a
// chunk are issued before its sums
template <int PL, int MV>
__device__ __forceinline__ void split_adc(const bool (&on)[PL], int rt, const uint8_t *s_stage, const float *s_tab,
                                          float (&acc)[PL]) {
    constexpr int M = 16 * MV;
    constexpr int CH = 16;  // table lookups issued ahead of their sums
#pragma unroll
    for (int r = 0; r < PL; ++r) {
        acc[r] = 0.0f;
        if (on[r]) {
            uint4 code[MV];
#pragma unroll
            for (int v = 0; v < MV; ++v)
                code[v] = *reinterpret_cast<const uint4 *>(s_stage + (rt + 64 * r) * M + 16 * v);
#pragma unroll
            for (int s0 = 0; s0 < M; s0 += CH) {
                float e[CH];
#pragma unroll
                for (int q = 0; q < CH; ++q) {
                    const int s = s0 + q;
                    const uint32_t word = u4_word(code[s >> 4], (s >> 2) & 3);
                    e[q] = s_tab[s * 256 + ((word >> (8 * (s & 3))) & 0xFFu)];
                }
#pragma unroll
                for (int q = 0; q < CH; ++q) acc[r] = __fadd_rn(acc[r], e[q]);
            }
        }
    }
}

// Row warps: the row of node w -> keys in s_key[0, 64*PL) (SENTINEL for
// slots past the degree and for neighbours the Bloom filter drops); their
// minimum and fresh count in s_m (parity `par`).  rt = thread index among
// the 64 row threads.

template <int PL, int MV>
__device__ __forceinline__ void split_row(const SearchParams &p, uint32_t w, int rt, const float *s_tab,
                                          uint32_t *bits, uint64_t *s_key, SplitMisc *s_m, int par,
                                          uint8_t *s_stage, uint8_t *s_tf, const int32_t *s_hrow, bool hop1) {
    constexpr int M = 16 * MV;
    const int rw = rt >> 5, lane = rt & 31;
    // (p.profile == 2) row thread 0's cycles from entry to each stage, per hop
    const bool bk = p.profile == 2 && rt == 0;
    const long long c0 = bk ? clock64() : 0;
#define SPLIT_STAMP(slot, dep) \
    if (bk) s_m->ph[slot] += (unsigned long long)(clock_after((int)(dep)) - c0);
    const int32_t *row = p.adj + (int64_t)w * p.adj_stride;
    uint32_t nid[PL];
    int deg;
    bool shared = true;  // in-row slot sharing at this z (unknown: the exact path)
    bool pre = false;
    // The list warps staged the published head's row ids + deg_share word
    // (68% of hops expand the old head): no adjacency read then.  Every hop
    // h >= 1 the row warps arrive on barrier 5 once they hold s_hrow, so the
    // list warps may overwrite it (they sync on 5 late in the hop).
    if (hop1 && p.head_row && p.deg_share && !p.host_graph) {
        uint32_t dep = 0;
        if (s_m->hid == w) {
            pre = true;
            const int32_t v = s_m->hdeg;
            deg = v & 0x7FFFFFFF;
            shared = v < 0;
#pragma unroll
            for (int r = 0; r < PL; ++r) {
                nid[r] = rt + 64 * r < p.R ? (uint32_t)s_hrow[rt + 64 * r] : 0u;
                dep ^= nid[r];
            }
        }
        asm volatile("bar.arrive 5, 128;" ::"r"(dep) : "memory");
    }
    if (pre) {
    } else
    if (p.deg_share) {
        // degree + sharing flag in one load (HBM; host-mapped rows too)
        const int32_t v = __ldg(p.deg_share + w);
        deg = v & 0x7FFFFFFF;
        shared = v < 0;
#pragma unroll
        for (int r = 0; r < PL; ++r)
            nid[r] = rt + 64 * r < p.R ? (uint32_t)(p.host_graph ? row[rt + 64 * r] : __ldg(row + rt + 64 * r)) : 0u;
    } else if (p.host_graph) {
        // pinned, mapped host rows read over PCIe; with a [deg, 0, 0, 0]
        // header (p.row_hdr) degree and ids come in one coalesced read
        deg = p.row_hdr ? row[-4] : p.deg[w];
#pragma unroll
        for (int r = 0; r < PL; ++r) nid[r] = rt + 64 * r < p.R ? (uint32_t)row[rt + 64 * r] : 0u;
    } else {
        deg = __ldg(p.deg + w);
#pragma unroll
        for (int r = 0; r < PL; ++r) nid[r] = rt + 64 * r < p.R ? (uint32_t)__ldg(row + rt + 64 * r) : 0u;
    }
    SPLIT_STAMP(0, nid[0] ^ (uint32_t)deg)
    uint32_t p1[PL], p2[PL];
    bool fresh[PL];
    float acc[PL];
    if (!shared) {
        // ---- no two probes of this row share a slot: batched test-then-set
        // equals sequential test-and-set (bloom.py:135-151) and each
        // fetch-or returns the pre-state of its own bits, so the sets go out
        // at once (no pre-state read, no row barrier; setting the bits of a
        // probe that turns out not fresh is a no-op -- both were set).  The
        // code rows are staged by cp.async meanwhile and every probe's ADC
        // runs while the fetch-ors return.
        bool on[PL];
#pragma unroll
        for (int r = 0; r < PL; ++r) {
            on[r] = rt + 64 * r < deg;
            p1[r] = p2[r] = 0u;
            if (on[r]) {
                p1[r] = mod_z(fnv1a(nid[r], kFnvOffset), p.geom);
                p2[r] = mod_z(fnv1a(nid[r], kFnvOffsetH2), p.geom);
                const uint8_t *crow = p.codes + (int64_t)nid[r] * p.code_stride;
#pragma unroll
                for (int v = 0; v < MV; ++v)
                    code_copy16(s_stage + (rt + 64 * r) * M + 16 * v, crow + 16 * v);
            }
        }
        __pipeline_commit();
        uint32_t o1[PL], o2[PL];
#pragma unroll
        for (int r = 0; r < PL; ++r) {
            o1[r] = o2[r] = 0u;
            // (O2COPY: o2 = o1 when the slots coincide.  The register move
            // waits for the fetch-or's round trip before the ADC starts, and
            // that measured 2% faster than deferring the wait:
            // profiles/r02/ab_v4/)
            if (on[r]) {
                o1[r] = bloom_or(bits + (p1[r] >> 5), 1u << (p1[r] & 31));
                o2[r] = p2[r] != p1[r] ? bloom_or(bits + (p2[r] >> 5), 1u << (p2[r] & 31)) : o1[r];
            }
        }
        SPLIT_STAMP(1, p1[0])
        __pipeline_wait_prior(0);  // this thread's own staged rows
        split_adc<PL, MV>(on, rt, s_stage, s_tab, acc);
        SPLIT_STAMP(3, __float_as_int(acc[0]))
#pragma unroll
        for (int r = 0; r < PL; ++r)
            fresh[r] = on[r] && !(((o1[r] >> (p1[r] & 31)) & 1u) &&
                                  (p2[r] == p1[r] || ((o2[r] >> (p2[r] & 31)) & 1u)));
        SPLIT_STAMP(5, fresh[0])
    } else {
    // ---- the Bloom slots and pre-state words (L2), then the code-row
    // gathers (HBM) staged into shared memory by cp.async.  The copies'
    // completion is tracked apart from the Bloom words', so the Bloom test
    // and the row's sets do not wait for HBM (issuing the copies first was
    // measured 7% slower: the Bloom words are the longer chain).
    uint32_t wd1[PL], wd2[PL];
#pragma unroll
    for (int r = 0; r < PL; ++r) {
        p1[r] = p2[r] = wd1[r] = wd2[r] = 0u;
        if (rt + 64 * r < deg) {
            p1[r] = mod_z(fnv1a(nid[r], kFnvOffset), p.geom);
            p2[r] = mod_z(fnv1a(nid[r], kFnvOffsetH2), p.geom);
            wd1[r] = bloom_ld(bits + (p1[r] >> 5));
            wd2[r] = bloom_ld(bits + (p2[r] >> 5));
        }
    }
#pragma unroll
    for (int r = 0; r < PL; ++r) {
        if (rt + 64 * r < deg) {
            const uint8_t *crow = p.codes + (int64_t)nid[r] * p.code_stride;
#pragma unroll
            for (int v = 0; v < MV; ++v)
                code_copy16(s_stage + (rt + 64 * r) * M + 16 * v, crow + 16 * v);
        }
    }
    __pipeline_commit();
    // ---- Bloom test against the pre-state (bloom.py:70-75 semantics)
    bool pf[PL], b1[PL], b2[PL];
#pragma unroll
    for (int r = 0; r < PL; ++r) {
        b1[r] = (wd1[r] >> (p1[r] & 31)) & 1u;
        b2[r] = (wd2[r] >> (p2[r] & 31)) & 1u;
        pf[r] = rt + 64 * r < deg && !(b1[r] && b2[r]);
    }
    SPLIT_STAMP(1, pf[0])
    if (rt == 0) s_m->coll = 0;
    // every row thread holds its pre-state words before any set of this row
    // lands (the words are consumed above)
    split_bar(3, 64);
    SPLIT_STAMP(2, 0)
    uint32_t o1[PL], o2[PL];
#pragma unroll
    for (int r = 0; r < PL; ++r) {
        o1[r] = o2[r] = 0u;
        if (pf[r]) {
            o1[r] = bloom_or(bits + (p1[r] >> 5), 1u << (p1[r] & 31));
            if (p2[r] != p1[r]) o2[r] = bloom_or(bits + (p2[r] >> 5), 1u << (p2[r] & 31));
        }
    }
    // ---- ADC of the presumed-fresh neighbours while the fetch-ors return
    __pipeline_wait_prior(0);  // this thread's own staged rows
    split_adc<PL, MV>(pf, rt, s_stage, s_tab, acc);
    SPLIT_STAMP(3, __float_as_int(acc[0]))
    // ---- in-row slot sharing: a fetch-or found its bit set although the
    // pre-state lacked it -> another probe of this row set it first
    bool sh1[PL], sh2[PL];
    bool any_sh = false;
#pragma unroll
    for (int r = 0; r < PL; ++r) {
        sh1[r] = pf[r] && !b1[r] && ((o1[r] >> (p1[r] & 31)) & 1u);
        sh2[r] = pf[r] && p2[r] != p1[r] && !b2[r] && ((o2[r] >> (p2[r] & 31)) & 1u);
        any_sh = any_sh || sh1[r] || sh2[r];
    }
    if (any_sh) s_m->coll = 1;
    split_bar(3, 64);
    SPLIT_STAMP(5, 0)
#pragma unroll
    for (int r = 0; r < PL; ++r) fresh[r] = pf[r];
    if (s_m->coll) {
        RowProbes<PL> pr;
        pr.pf = pr.b1 = pr.b2 = pr.sh1 = pr.sh2 = 0;
#pragma unroll
        for (int r = 0; r < PL; ++r) {
            pr.p1[r] = p1[r];
            pr.p2[r] = p2[r];
            pr.pf |= (uint32_t)pf[r] << r;
            pr.b1 |= (uint32_t)b1[r] << r;
            pr.b2 |= (uint32_t)b2[r] << r;
            pr.sh1 |= (uint32_t)sh1[r] << r;
            pr.sh2 |= (uint32_t)sh2[r] << r;
        }
        const uint32_t f = split_replay<PL>(rt, deg, pr, s_stage, bits, s_tf);
#pragma unroll
        for (int r = 0; r < PL; ++r) fresh[r] = (f >> r) & 1u;
    }
    }
    // keys out; per-warp minimum (dist bits, then id: two 32-bit
    // reductions) and fresh count
    int fc = 0;
    uint64_t mn = kSentinel;
#pragma unroll
    for (int r = 0; r < PL; ++r) {
        const uint64_t key = fresh[r] ? pack_key(acc[r], nid[r]) : kSentinel;
        s_key[rt + 64 * r] = key;
        mn = key < mn ? key : mn;
        fc += fresh[r];
    }
    const uint32_t mhi = __reduce_min_sync(kFull, (uint32_t)(mn >> 32));
    const uint32_t mlo = __reduce_min_sync(kFull, (uint32_t)(mn >> 32) == mhi ? (uint32_t)mn : 0xFFFFFFFFu);
    fc = __reduce_add_sync(kFull, fc);
    const uint64_t wmin = ((uint64_t)mhi << 32) | mlo;
    if (lane == 0) {
        s_m->rmin[par][rw] = wmin;
        s_m->rfresh[par][rw] = fc;
    }
    if (rt == 0) s_m->rdeg[par] = deg;
    SPLIT_STAMP(6, fc)
#undef SPLIT_STAMP
}

// List warps: merge the survivors of s_key (keys < thr) into the worklist
// (kernels.py:68-87: rank of each entry in the other list, old entries first
// on ties -- keys are unique), mark the winner visited and log it, publish
// the next head / threshold / count at parity `nxt`.  lt = thread index
// among the 64 list threads.  s_c (t int16): survivors below each old entry;
// s_spos (RPAD int16): final position of each sorted survivor.
template <int PL>
__device__ __forceinline__ void split_list(const SearchParams &p, int lt, uint64_t *s_wl, uint8_t *s_vis,
                                           const uint64_t *s_key, uint64_t *s_nk, uint64_t *s_sk, int16_t *s_c,
                                           int16_t *s_spos, SplitMisc *s_m, int nxt, uint64_t winner,
                                           uint64_t head, uint64_t thr, int cnt, int hpos, int32_t *log, int iters,
                                           int32_t *s_hrow) {
    constexpr int NC = 64;      // list threads
    constexpr int MAXCH = 4;    // worklists up to 4*NC entries (checked on the host)
    constexpr int H = 32 * PL;  // survivors region per list warp
    const int lane = lt & 31, lw = lt >> 5;
    const int t = p.t;
    const unsigned ltm = (1u << lane) - 1u;
    const bool won_head = winner == head;
    // (p.profile == 3) list thread 0's cycles from entry to each stage, per hop
    const bool bk = p.profile == 3 && lt == 0;
    const long long c0 = bk ? clock64() : 0;
#define SPLIT_STAMP(slot, dep) \
    if (bk) s_m->ph[slot] += (unsigned long long)(clock_after((int)(dep)) - c0);
    // ---- survivors (keys < thr: ranks >= t are truncated, engine.py:213)
    // compacted per list warp in adjacency order
    uint64_t k[PL];
    bool sv[PL];
    int cw = 0;
#pragma unroll
    for (int r = 0; r < PL; ++r) {
        k[r] = s_key[lt + 64 * r];
        sv[r] = k[r] < thr;
        const unsigned b = __ballot_sync(kFull, sv[r]);
        if (sv[r]) s_nk[H * lw + cw + __popc(b & ltm)] = k[r];
        cw += __popc(b);
    }
    if (lane == 0) s_m->wsurv[lw] = cw;
    // the next unvisited old entry after the winner: the old head itself, or
    // (the head won) the first unvisited entry after it
    if (lw == 0) {
        const int op = won_head ? first_unvisited(s_vis, hpos + 1, cnt) : hpos;
        if (lane == 0) {
            s_m->opos = op;
            s_m->okey = op < cnt ? s_wl[op] : kSentinel;
        }
    }
    split_bar(4, NC);
    const int c0w = s_m->wsurv[0], c1w = s_m->wsurv[1];
    const int n = c0w + c1w;
    SPLIT_STAMP(0, n)
    // ---- kernels 4a + 4b in one pass over the (unsorted) survivors, from
    // the same broadcast reads: each survivor's rank among them (its sorted
    // slot) and each old entry's count of smaller survivors (keys are unique)
    const int nch = (cnt + NC - 1) / NC;
    uint64_t mv[MAXCH];
    uint8_t mvv[MAXCH];
    int mc[MAXCH];
#pragma unroll
    for (int c = 0; c < MAXCH; ++c) {
        const int i = c * NC + lt;
        mv[c] = kSentinel;
        mvv[c] = 0;
        mc[c] = 0;
        if (c < nch && i < cnt) {
            mv[c] = s_wl[i];
            mvv[c] = s_vis[i];
        }
    }
    if (n > 0) {
        int rk[PL];
#pragma unroll
        for (int r = 0; r < PL; ++r) rk[r] = 0;
        auto count = [&](const uint64_t sk) {
#pragma unroll
            for (int r = 0; r < PL; ++r) rk[r] += sk < k[r];
#pragma unroll
            for (int c = 0; c < MAXCH; ++c) mc[c] += sk < mv[c];
        };
        for (int i = 0; i < c0w; ++i) count(s_nk[i]);
        for (int i = 0; i < c1w; ++i) count(s_nk[H + i]);
#pragma unroll
        for (int r = 0; r < PL; ++r)
            if (sv[r]) s_sk[rk[r]] = k[r];
#pragma unroll
        for (int c = 0; c < MAXCH; ++c)
            if (c < nch && c * NC + lt < cnt) s_c[c * NC + lt] = (int16_t)mc[c];
    }
    SPLIT_STAMP(1, 0)
    SPLIT_STAMP(2, mc[0])
    split_bar(4, NC);  // all reads of the old worklist precede the writes
    // ---- merge + truncate to t (engine.py:210-215): old entry i goes to
    // i + c_i; survivors c_{i-1} .. c_i - 1 land just before it, the rest
    // after the last old entry
    if (n > 0) {
#pragma unroll
        for (int c = 0; c < MAXCH; ++c) {
            const int i = c * NC + lt;
            if (c < nch && i < cnt) {
                const int ci = mc[c];
                const int prev = i > 0 ? s_c[i - 1] : 0;
                if (i + ci < t) {
                    s_wl[i + ci] = mv[c];
                    s_vis[i + ci] = mvv[c];
                }
                for (int r = prev; r < ci; ++r) {
                    s_spos[r] = (int16_t)(i + r);
                    if (i + r < t) {
                        s_wl[i + r] = s_sk[r];
                        s_vis[i + r] = 0;
                    }
                }
                if (i == cnt - 1)
                    for (int r = ci; r < n; ++r) {
                        s_spos[r] = (int16_t)(cnt + r);
                        if (cnt + r < t) {
                            s_wl[cnt + r] = s_sk[r];
                            s_vis[cnt + r] = 0;
                        }
                    }
            }
        }
    }
    const int ncnt = min(t, cnt + n);
    split_bar(4, NC);  // the merged worklist is complete
    SPLIT_STAMP(3, 0)
    // ---- expand the winner (engine.py:167-178); the next head is the
    // smaller of the next old unvisited entry and the best survivor other
    // than the winner, at its merged position (none if truncated)
    if (lt == 0) {
        // loads first (the stores below may alias them for the compiler)
        const int op = s_m->opos;
        uint64_t hk = s_m->okey;
        const int rs = won_head ? 0 : 1;  // best survivor other than the winner
        const int c_h = n > 0 && won_head ? s_c[hpos] : 0;
        const int c_o = n > 0 && op < cnt ? s_c[op] : 0;
        const int sp0 = n > 0 ? s_spos[0] : 0;
        const uint64_t skr = rs < n ? s_sk[rs] : kSentinel;
        const int spr = rs < n ? s_spos[rs] : t;
        const uint64_t last = s_wl[t - 1];
        const int wpos = won_head ? hpos + c_h : sp0;
        if (p.debug && (wpos >= t || s_wl[wpos] != winner)) atomicAdd(p.counters + kCtrDebugFail, 1ull);
        int hp = op < cnt ? op + c_o : t;
        if (skr < hk) {
            hk = skr;
            hp = spr;
        }
        if (hp >= ncnt) {
            hk = kSentinel;
            hp = ncnt;
        }
        if (wpos < t) s_vis[wpos] = 1;
        if (iters < p.log_cap) log[iters] = (int32_t)key_id(winner);
        s_m->hpos[nxt] = hp;
        s_m->head[nxt] = hk;
        s_m->thr[nxt] = ncnt == t ? last : kSentinel;
        s_m->cnt[nxt] = ncnt;
        // the head may be the next winner: its row to L2
        if (p.row_prefetch && hk != kSentinel) prefetch_row_l2(p, key_id(hk));
    }
    // stage the published head's row ids + deg_share word for the row warps
    // (used when it wins the next hop); the loads run in the list warps'
    // slack before the hop barrier
    if (p.head_row && p.deg_share && !p.host_graph) {
        split_bar(4, NC);  // the published head
        const uint64_t hk2 = s_m->head[nxt];
        int32_t ids[PL];
        int32_t hv = 0;
        uint32_t hid = 0xFFFFFFFFu;
#pragma unroll
        for (int r = 0; r < PL; ++r) ids[r] = 0;
        if (hk2 != kSentinel) {
            hid = key_id(hk2);
            const int32_t *hrow = p.adj + (int64_t)hid * p.adj_stride;
#pragma unroll
            for (int r = 0; r < PL; ++r)
                if (lt + 64 * r < p.R) ids[r] = __ldg(hrow + lt + 64 * r);
            if (lt == 0) hv = __ldg(p.deg_share + hid);
        }
        split_bar(5, 128);  // the row warps hold this hop's s_hrow
#pragma unroll
        for (int r = 0; r < PL; ++r) s_hrow[lt + 64 * r] = ids[r];
        if (lt == 0) {
            s_m->hdeg = hv;
            s_m->hid = hid;
        }
    }
    SPLIT_STAMP(4, 0)
    if (bk) {  // hop statistics: expansions of the old head, survivors merged
        s_m->ph[5] += won_head;
        s_m->ph[6] += (unsigned long long)n;
    }
#undef SPLIT_STAMP
}

// Per-query prologue (all 128 threads): the query, the cleared filter
// (whole-line stores), kernel 1 into shared memory (pq.py:284-296) and the
// medoid in the filter (engine.py:127-128).  (Measured 2% faster inline than
// out of line.)
template <int SUB, int MV>
__device__ __forceinline__ void split_prologue(const SearchParams &p, int64_t qid, float *s_q, uint8_t *s_vis,
                                            float *s_tab, uint32_t *bits) {
    constexpr int NT = 128;
    constexpr int M = 16 * MV;
    const int tid = threadIdx.x;
    // parameters in registers: through the generic pointer the compiler must
    // assume the shared-memory stores below may alias them
    const int dim = p.dim, t = p.t;
    const float *__restrict__ queries = p.queries;
    const float *__restrict__ centroids = p.centroids;
    const int32_t *__restrict__ sub_off = p.sub_off;
    const int32_t *__restrict__ sub_size = p.sub_size;
    const int n4 = (int)(p.bloom_stride >> 2);
    const uint32_t mp1 = p.medoid_p1, mp2 = p.medoid_p2;
    for (int i = tid; i < dim; i += NT) s_q[i] = __ldg(queries + qid * dim + i);
    for (int i = tid; i < t; i += NT) s_vis[i] = 0;
    {   // the filter starts empty (whole-line stores)
        uint4 *b4 = reinterpret_cast<uint4 *>(bits);
        for (int i = tid; i < n4; i += NT) bloom_st4(b4 + i, make_uint4(0u, 0u, 0u, 0u));
    }
    __syncthreads();
    // kernel 1 for this query into shared memory (pq.py:284-296); the
    // centroid loads (L2) of 8 entries per thread are in flight together
#pragma unroll kTabUnroll
    for (int idx = tid; idx < M * 256; idx += NT) {
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
            float a = __fmul_rn(dd, dd);
            for (int q = 1; q < sz; ++q) {
                dd = __fsub_rn(s_q[off + q], __ldg(src + q));
                a = __fadd_rn(a, __fmul_rn(dd, dd));
            }
            e = a;
        }
        s_tab[idx] = e;
    }
    if (tid == 0) {  // the medoid in the filter (engine.py:127-128)
        const uint32_t w1 = mp1 >> 5, w2 = mp2 >> 5;
        const uint32_t b1 = 1u << (mp1 & 31), b2 = 1u << (mp2 & 31);
        if (w1 == w2) {
            bloom_st(bits + w1, b1 | b2);
        } else {
            bloom_st(bits + w1, b1);
            bloom_st(bits + w2, b2);
        }
    }
    __syncthreads();
}

// Per-query epilogue (engine.py:244-269): re-rank of the visit
// log (kernel 5) with the rows staged through the dead table and the keys
// kept in shared memory for the top-k, or the worklist's first k without
// re-rank.  Returns the re-ranked candidates (thread 0), 0 if the log
// overflowed (the host re-runs the query).
template <int MV>
__device__ __forceinline__ int split_epilogue(const SearchParams &p, int64_t qid, int iters, int cnt,
                                           const int32_t *log, const float *s_q, const uint64_t *s_wl,
                                           float *s_tab, uint64_t *rr) {
    constexpr int M = 16 * MV;
    const int tid = threadIdx.x;
    int32_t *oid = p.out_ids + qid * p.k;
    float *odist = p.out_dists + qid * p.k;
    if (tid == 0) {
        p.out_iters[qid] = iters;
        p.out_wall_ns[qid] = globaltimer_ns() - p.counters[kCtrT0];
    }
    if (!p.rerank) {
        if (p.log_cap < iters && tid == 0) {
            const unsigned long long at = atomicAdd(p.counters + kCtrOverflow, 1ull);
            p.overflow_list[at] = (int32_t)qid;
        }
        for (int q = tid; q < p.k; q += 128) {
            if (q < cnt) {
                oid[q] = (int32_t)key_id(s_wl[q]);
                odist[q] = key_dist(s_wl[q]);
            } else {
                oid[q] = -1;
                odist[q] = __int_as_float(0x7f800000);
            }
        }
        if (tid == 0) p.out_short[qid] = cnt < p.k;
        return 0;
    }
    if (iters > p.log_cap) {  // visit log truncated: the host re-runs this query
        if (tid == 0) {
            const unsigned long long at = atomicAdd(p.counters + kCtrOverflow, 1ull);
            p.overflow_list[at] = (int32_t)qid;
        }
        return 0;
    }
    // kernel 5: exact distances of the visit log, then top-k (warp 0)
    __threadfence_block();
    __syncthreads();
    const int rowb = p.dim * (p.vec_dtype == kVecF32 ? 4 : 1);
    const int tab_b = M * 256 * 4, kb = (8 * iters + 15) & ~15;
    if (rowb % 16 == 0 && kb <= tab_b / 2 && rowb <= tab_b - kb) {
        // the table is dead until the next query: stage rows in its place and
        // keep the keys at its end, so the top-k reads shared memory
        uint64_t *s_rr = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(s_tab) + tab_b - kb);
        rerank_staged<128>(p, log, iters, s_q, reinterpret_cast<uint8_t *>(s_tab), tab_b - kb, s_rr);
        if (tid < 32) {
            warp_topk_write_smem(s_rr, iters, p.k, oid, odist);
            if (tid == 0) p.out_short[qid] = iters < p.k;
        }
        return tid == 0 ? iters : 0;
    }
    for (int i = tid; i < iters; i += 128) {
        const uint32_t node = (uint32_t)__ldcg(log + i);
        rr[i] = pack_key(exact_sq_dist(p.vectors, p.vec_dtype, p.dim, node, s_q), node);
    }
    __threadfence_block();
    __syncthreads();
    if (tid < 32) {
        warp_topk_write(rr, iters, p.k, oid, odist);
        if (tid == 0) p.out_short[qid] = iters < p.k;
    }
    return tid == 0 ? iters : 0;
}

template <int PL, int SUB, int MV>
__global__ void __launch_bounds__(128, MV == 3 ? 4 : 5) search_split_kernel(const __grid_constant__ SearchParams p) {
    constexpr int M = 16 * MV;
    constexpr int RPAD = 64 * PL;
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x;
    const bool roww = tid < 64;  // row warps 0-1, list warps 2-3

    float *s_q = reinterpret_cast<float *>(smem + p.off_q);
    uint64_t *s_wl = reinterpret_cast<uint64_t *>(smem + p.off_wl);
    uint64_t *s_sk = reinterpret_cast<uint64_t *>(smem + p.off_sk);
    uint64_t *s_nk = reinterpret_cast<uint64_t *>(smem + p.off_nk);
    uint64_t *s_key = reinterpret_cast<uint64_t *>(smem + p.off_code);  // [2][RPAD]
    int16_t *s_c = reinterpret_cast<int16_t *>(smem + p.off_fid);          // [t]
    int16_t *s_spos = s_c + ((p.t + 7) & ~7);                              // [RPAD]
    uint8_t *s_stage = smem + p.off_dup;  // [RPAD][M] staged code rows / replay records
    uint8_t *s_tf = smem + p.off_alive;                                   // [RPAD]
    int32_t *s_hrow = reinterpret_cast<int32_t *>(smem + p.off_hrow);     // [RPAD] staged head row
    uint8_t *s_vis = smem + p.off_vis;
    float *s_tab = reinterpret_cast<float *>(smem + p.off_tab);
    SplitMisc *s_m = reinterpret_cast<SplitMisc *>(smem + p.off_acc);
    uint32_t *bits = p.bloom + (int64_t)blockIdx.x * p.bloom_stride;
    uint64_t *rr = p.rr_scratch + (int64_t)blockIdx.x * p.log_cap;
    const int t = p.t;

    unsigned long long st_iters = 0, st_probes = 0, st_fresh = 0, st_rr = 0;
    // phase profiler (p.profile): 0 row chain (row thread 0), 1 list step
    // (list thread 0), 2/3 their waits at the hop barrier, 7 per-query prologue
    // + epilogue (thread 0)
    if (tid == 0)
        for (int i = 0; i < 8; ++i) s_m->ph[i] = 0;
    const bool prof = p.profile == 1 && (tid == 0 || tid == 64);

    for (;;) {
        long long c_q = p.profile ? clock64() : 0;
        if (tid == 0) s_m->qi = (long long)atomicAdd(p.counters + kCtrNextQuery, 1ull);
        __syncthreads();
        const int64_t qi = s_m->qi;
        if (qi >= p.nq) break;
        const int64_t qid = p.query_map ? (int64_t)p.query_map[qi] : qi;

        split_prologue<SUB, MV>(p, qid, s_q, s_vis, s_tab, bits);
        int32_t *log = p.visit_log + (p.query_map ? qi : qid) * p.log_cap;
        if (tid == 64) {
            // worklist = [key(ADC(medoid), medoid)] (engine.py:118-125), expanded at once
            const uint8_t *row = p.codes + (int64_t)p.medoid * p.code_stride;
            float acc = 0.0f;
            for (int s = 0; s < M; ++s) acc = __fadd_rn(acc, s_tab[s * 256 + __ldg(row + s)]);
            s_wl[0] = pack_key(acc, (uint32_t)p.medoid);
            s_vis[0] = 1;
            if (p.log_cap > 0) log[0] = p.medoid;
            s_m->head[0] = kSentinel;
            s_m->hpos[0] = 1;
            s_m->thr[0] = t == 1 ? s_wl[0] : kSentinel;
            s_m->cnt[0] = 1;
            s_m->hid = 0xFFFFFFFFu;
        }
        if (p.profile && tid == 0) {
            const long long now_ = clock64();
            s_m->ph[7] += (unsigned long long)(now_ - c_q);
        }
        __syncthreads();

        // hop 0 is the medoid's row (row warps only, written at parity 0);
        // hop h >= 1 expands the eager winner chosen at its barrier.  One
        // call site per role keeps the hop loop's code compact.
        int iters = 0, par = 1;
        for (;;) {
            uint64_t winner, head = kSentinel, thr = kSentinel;
            if (iters == 0) {
                winner = (uint64_t)(uint32_t)p.medoid;
            } else {
                // ---- the hop barrier: eager winner and convergence (engine.py:201-217)
                const uint64_t rmin = min(s_m->rmin[par][0], s_m->rmin[par][1]);
                head = s_m->head[par];
                thr = s_m->thr[par];
                winner = rmin < head ? rmin : head;
                st_probes += s_m->rdeg[par];
                st_fresh += s_m->rfresh[par][0] + s_m->rfresh[par][1];
                if (head == kSentinel && !(rmin < thr)) break;  // merged worklist all visited
            }
            const long long c0 = prof ? clock64() : 0;
            if (roww) {
                split_row<PL, MV>(p, key_id(winner), tid, s_tab, bits, s_key + (par ^ 1) * RPAD, s_m, par ^ 1,
                                  s_stage, s_tf, s_hrow, iters > 0);
            } else if (iters > 0) {
                split_list<PL>(p, tid - 64, s_wl, s_vis, s_key + par * RPAD, s_nk, s_sk, s_c, s_spos, s_m, par ^ 1,
                               winner, head, thr, s_m->cnt[par], s_m->hpos[par], log, iters, s_hrow);
            }
            long long c1 = 0;
            if (prof) {
                c1 = clock64();
                s_m->ph[tid == 0 ? 0 : 1] += (unsigned long long)(c1 - c0);
            }
            ++iters;
            par ^= 1;
            __syncthreads();
            if (prof) s_m->ph[tid == 0 ? 2 : 3] += (unsigned long long)(clock_after(s_m->cnt[par]) - c1);
        }
        st_iters += iters;
        c_q = p.profile ? clock64() : 0;

        // ---- outputs (engine.py:244-269)
        st_rr += split_epilogue<MV>(p, qid, iters, s_m->cnt[par], log, s_q, s_wl, s_tab, rr);
        __syncthreads();
        if (p.profile && tid == 0) s_m->ph[7] += (unsigned long long)(clock64() - c_q);
    }
    if (p.profile && tid == 0) {
        __syncwarp();
        // slots written by row thread 0 / list thread 0 of this CTA; all
        // writers are past the CTA's last barrier
#pragma unroll
        for (int i = 0; i < 8; ++i) atomicAdd(p.counters + kCtrPhase0 + i, s_m->ph[i]);
    }
    if (tid == 0) {
        atomicAdd(p.counters + kCtrIterations, st_iters);
        atomicAdd(p.counters + kCtrRerank, st_rr);
        atomicAdd(p.counters + kCtrProbes, st_probes);
        atomicAdd(p.counters + kCtrFresh, st_fresh);
    }
}

}  // namespace bang
