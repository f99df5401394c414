// bang_search_pf.cuh -- search_cta_kernel with the next row's memory phase
// taken off the critical path (the paper's "one hop ahead" prefetch,
// PAPER.md:922-938, carried to the Bloom words and code rows).
//
// As soon as the eager winner is known (engine.py:201-205) the prefetch warps
// (1 or 2, PFW) leave the iteration's sort + merge to the other warps and, for
// the winner's adjacency row,
//   * load the neighbour ids and the degree (the candidate winners' rows were
//     already asked of L2 at expand / survivor time),
//   * hash every id into its two Bloom slots (bloom.py:26-42) and read the
//     slots' pre-state bits -- every set of this row is already performed
//     (the fetch-or results were consumed before the collision barrier),
//   * stage the neighbours' PQ code rows into shared memory with cp.async
//     (or, when they do not fit, ask L2 for them),
// and leave ids, slots, bits and codes in shared memory.  The next iteration
// then starts from shared memory only: no global load precedes its Bloom test
// or its ADC.  Everything else -- table, ADC, exact in-row collision replay,
// sort, merge, convergence, re-rank -- is search_cta_kernel's, bit for bit
// (SURVEY.md 8(a0)).
//
// Filters are cleared with whole-line stores at query start, so every probe
// reads its word (no summary bitmap; its shared memory holds the staged rows).
#pragma once

#include "bang_search_cta.cuh"

namespace bang {

struct PfMisc {
    unsigned long long wmin[8];  // per-warp survivor minimum
    int wcnt[8];                 // per-warp survivor count
    int wfresh[8];               // per-warp fresh count
    long long qi;
    int hpos;
    int wpos;
    unsigned long long head;
    unsigned long long ph[8];  // phase profiler: thread 32's cycles per phase
    long long t_ph;
    int ndeg;                  // degree of the prefetched row
};
static_assert(sizeof(PfMisc) <= 256, "PfMisc must fit its 256-byte smem slot");

__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void l2_prefetch(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p) : "memory");
}
// adjacency row + degree of node v towards L2 (speculative: a candidate for
// the next winner, PAPER.md:922-938 one hop ahead)
__device__ __forceinline__ void prefetch_row_l2(const SearchParams &p, uint32_t v) {
    const int32_t *row = p.adj + (int64_t)v * p.adj_stride;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(row) : "memory");
    if (((uintptr_t)row & 127u) + 4u * (uint32_t)p.R > 128u)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(row + p.R - 1) : "memory");
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p.deg + v) : "memory");
}
// clock64 read that waits for v (a value loaded after a barrier): a barrier
// blocks only at the first use of what it protects, so the profiler's clock
// must depend on such a use
__device__ __forceinline__ long long clock_after(int v) {
    long long c;
    asm volatile("{\n\t.reg .u32 t;\n\tmov.u32 t, %1;\n\tmov.u64 %0, %%clock64;\n\t}" : "=l"(c) : "r"(v) : "memory");
    return c;
}

// Warp 0: the row of node w -> s_nid (ids), s_nps (slot per probe half),
// s_nfl (bit0 = pre-state bit, bit1 = word marked in the summary), ndeg; the
// code rows are prefetched into L2.
template <int NT, int MV, int PFW>
__device__ __forceinline__ void pf_row(const SearchParams &p, uint32_t w, int lane, uint8_t *s_code,
                                       const uint32_t *bits, uint32_t *s_nid, uint32_t *s_nps,
                                       uint8_t *s_nfl, PfMisc *s_m) {
    constexpr int PL = NT / (64 * PFW);  // neighbour slots per lane (RPAD = NT/2 over PFW warps)
    constexpr int PT = 32 * PFW;         // prefetch threads; lane = index among them
    constexpr int M = 16 * MV;
    const long long c0 = p.profile == 2 ? clock64() : 0;
    if (p.profile == 2)  // (breakdown) the row loads issue after c0
        asm volatile("mov.b32 %0, %0;" : "+r"(w) : "l"(c0));
    const int deg = p.deg[w];
    uint32_t nid[PL];
#pragma unroll
    for (int r = 0; r < PL; ++r) {
        const int jj = lane + PT * r;
        nid[r] = jj < p.R ? (uint32_t)p.adj[(int64_t)w * p.adj_stride + jj] : 0u;
    }
    if (p.profile == 2 && lane == 0) {  // (breakdown) row arrival
        uint32_t x = nid[0];
#pragma unroll
        for (int r = 1; r < PL; ++r) x ^= nid[r];
        s_m->ph[4] += (unsigned long long)(clock_after((int)x + deg) - c0);
    }
    uint32_t ps1[PL], ps2[PL], wd1[PL], wd2[PL];
    bool i1[PL], i2[PL];
#pragma unroll
    for (int r = 0; r < PL; ++r) {
        const int jj = lane + PT * r;
        ps1[r] = ps2[r] = wd1[r] = wd2[r] = 0u;
        i1[r] = i2[r] = false;
        if (jj < deg) {
            const uint8_t *crow = p.codes + (int64_t)nid[r] * p.code_stride;
            if (p.pf_stage) {
#pragma unroll
                for (int v = 0; v < MV; ++v) __pipeline_memcpy_async(s_code + jj * M + v * 16, crow + v * 16, 16);
            } else {
                l2_prefetch(crow);
                if (((uintptr_t)crow & 31u) + M > 32u) l2_prefetch(crow + M - 1);
            }
            ps1[r] = mod_z(fnv1a(nid[r], kFnvOffset), p.geom);
            ps2[r] = mod_z(fnv1a(nid[r], kFnvOffsetH2), p.geom);
            // the filter was cleared at query start: every word is current
            i1[r] = i2[r] = true;
            wd1[r] = __ldcg(bits + (ps1[r] >> 5));
            wd2[r] = __ldcg(bits + (ps2[r] >> 5));
        }
    }
    if (p.profile == 2 && lane == 0) {  // (breakdown) hashes + Bloom word arrival
        uint32_t x = 0;
#pragma unroll
        for (int r = 0; r < PL; ++r) x ^= wd1[r] ^ wd2[r];
        s_m->ph[5] += (unsigned long long)(clock_after((int)x) - c0);
    }
    bool sh1[PL], sh2[PL];
#pragma unroll
    for (int r = 0; r < PL; ++r) sh1[r] = sh2[r] = false;
    // early Bloom sets (p.pf_early): the row's presumed-fresh probes set their
    // bits now, one iteration ahead of their test (the test reads the
    // pre-state bits above, and no other row of this query runs in between).
    // A fetch-or that finds its bit set though the pre-state did not have it
    // marks in-row slot sharing for the exact replay -- the same evidence the
    // compute threads' fetch-or gave, without its round trip on their path.
    if (p.pf_early) {
        uint32_t o1[PL], o2[PL];
        bool fr[PL];
#pragma unroll
        for (int r = 0; r < PL; ++r) {
            const uint32_t b1 = (wd1[r] >> (ps1[r] & 31)) & 1u, b2 = (wd2[r] >> (ps2[r] & 31)) & 1u;
            fr[r] = lane + PT * r < deg && !(b1 && b2);  // (consumes this thread's word loads)
        }
        // every prefetch lane holds its pre-state words before any set of the
        // row lands (lanes of one warp are not ordered without the warp barrier)
        if (PFW > 1) named_bar_sync(3, PT);
        else __syncwarp();
#pragma unroll
        for (int r = 0; r < PL; ++r) {
            o1[r] = o2[r] = 0u;
            if (fr[r]) {
                o1[r] = atomicOr(const_cast<uint32_t *>(bits) + (ps1[r] >> 5), 1u << (ps1[r] & 31));
                if (ps2[r] != ps1[r]) o2[r] = atomicOr(const_cast<uint32_t *>(bits) + (ps2[r] >> 5), 1u << (ps2[r] & 31));
            }
        }
#pragma unroll
        for (int r = 0; r < PL; ++r) {
            const uint32_t b1 = (wd1[r] >> (ps1[r] & 31)) & 1u, b2 = (wd2[r] >> (ps2[r] & 31)) & 1u;
            sh1[r] = fr[r] && !b1 && ((o1[r] >> (ps1[r] & 31)) & 1u);
            sh2[r] = fr[r] && ps2[r] != ps1[r] && !b2 && ((o2[r] >> (ps2[r] & 31)) & 1u);
        }
    }
#pragma unroll
    for (int r = 0; r < PL; ++r) {
        const int jj = lane + PT * r;
        s_nid[jj] = nid[r];
        s_nps[2 * jj] = ps1[r];
        s_nps[2 * jj + 1] = ps2[r];
        s_nfl[2 * jj] = (uint8_t)(((wd1[r] >> (ps1[r] & 31)) & 1u) | (i1[r] ? 2u : 0u) | (sh1[r] ? 4u : 0u));
        s_nfl[2 * jj + 1] = (uint8_t)(((wd2[r] >> (ps2[r] & 31)) & 1u) | (i2[r] ? 2u : 0u) | (sh2[r] ? 4u : 0u));
    }
    if (lane == 0) s_m->ndeg = deg;
    if (p.pf_stage) {
        __pipeline_commit();
        __pipeline_wait_prior(0);  // staged rows land before the iteration's barrier
    }
}

// STAGE: the next row's code rows are staged in smem (p.pf_stage); a template
// parameter so the staged instance has no global code-load path whose
// scoreboard the compiler could merge with the fetch-or's
template <int NT, int SUB, int MV, int PFW, bool STAGE>
__global__ void __launch_bounds__(NT, (MV == 3 ? 512 : 768) / NT) search_pf_kernel(const SearchParams p) {
    constexpr int NW = NT / 32;
    constexpr int NC = NT - 32 * PFW;  // sort/merge threads (warps PFW..)
    constexpr int M = 16 * MV;
    constexpr int MH = M / 2;       // subspaces per half
    constexpr int MHW = MH / 4;     // code words (u32) per half
    constexpr int RPAD = NT / 2;    // neighbour slots
    constexpr int MAXCH = 4;        // worklists up to 4*NC entries (checked on the host)
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int j = tid >> 1, h = tid & 1;
    const int tc = tid - 32 * PFW;  // index among the sort/merge threads
    const bool pfw = warp < PFW;    // a prefetch warp
    const unsigned lt = (1u << lane) - 1u;

    float *s_q = reinterpret_cast<float *>(smem + p.off_q);
    uint64_t *s_wl = reinterpret_cast<uint64_t *>(smem + p.off_wl);
    uint64_t *s_sk = reinterpret_cast<uint64_t *>(smem + p.off_sk);
    uint64_t *s_nk = reinterpret_cast<uint64_t *>(smem + p.off_nk);
    uint32_t *s_nid = reinterpret_cast<uint32_t *>(smem + p.off_fid);
    uint8_t *s_fl = smem + p.off_alive;
    uint8_t *s_vis = smem + p.off_vis;
    float *s_tab = reinterpret_cast<float *>(smem + p.off_tab);
    uint8_t *s_code = smem + p.off_code;  // next row's code rows (pf_stage)
    uint32_t *s_nps = reinterpret_cast<uint32_t *>(smem + p.off_dup);
    uint8_t *s_nfl = smem + p.off_dup + 4 * NT;
    PfMisc *s_m = reinterpret_cast<PfMisc *>(smem + p.off_acc);
    uint32_t *bits = p.bloom + (int64_t)blockIdx.x * p.bloom_stride;
    uint64_t *rr = p.rr_scratch + (int64_t)blockIdx.x * p.log_cap;
    const int t = p.t;

    unsigned long long st_iters = 0, st_probes = 0, st_fresh = 0, st_rr = 0;
    // phase profiler: thread 32 (a sort/merge thread) per phase; slot 1 =
    // thread 0's cycles in the one-hop-ahead prefetch
    const bool prof = p.profile && tc == 0;
    if (tc == 0)
        for (int i = 0; i < 8; ++i) s_m->ph[i] = 0;
#define BANG_PF_PHASE(i)                                       \
    if (prof) {                                                \
        const long long now_ = clock64();                      \
        s_m->ph[i] += (unsigned long long)(now_ - s_m->t_ph);  \
        s_m->t_ph = now_;                                      \
    }

    for (;;) {
        if (prof) s_m->t_ph = clock64();
        if (tid == 0) s_m->qi = (long long)atomicAdd(p.counters + kCtrNextQuery, 1ull);
        __syncthreads();
        const int64_t qi = s_m->qi;
        if (qi >= p.nq) break;
        const int64_t qid = p.query_map ? (int64_t)p.query_map[qi] : qi;

        for (int i = tid; i < p.dim; i += NT) s_q[i] = __ldg(p.queries + qid * p.dim + i);
        for (int i = tid; i < t; i += NT) s_vis[i] = 0;
        {   // the filter starts empty (whole-line stores)
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
        }
        __syncthreads();
        if (tid == 0) {  // worklist = [key(ADC(medoid), medoid)] (engine.py:118-125)
            const uint8_t *row = p.codes + (int64_t)p.medoid * p.code_stride;
            float acc = 0.0f;
            for (int s = 0; s < M; ++s) acc = __fadd_rn(acc, s_tab[s * 256 + __ldg(row + s)]);
            s_wl[0] = pack_key(acc, (uint32_t)p.medoid);
        }
        if (pfw) pf_row<NT, MV, PFW>(p, (uint32_t)p.medoid, tid, s_code, bits, s_nid, s_nps, s_nfl, s_m);
        int cnt = 1, upos = 0;
        uint32_t u = (uint32_t)p.medoid;
        int32_t *log = p.visit_log + (p.query_map ? qi : qid) * p.log_cap;
        int iters = 0;
        // ---- expand u (engine.py:163-178) by the first sort/merge warp: mark
        // it visited, log it, find the next unvisited entry (the eager head)
        // and start the head's row towards L2.  In the loop this runs at the
        // end of the merge, before the iteration's last barrier.
        auto expand = [&](int up, uint32_t uu, int cnt_, int it_) {
            if (lane == 0) {
                if (p.debug && key_id(s_wl[up]) != uu) atomicAdd(p.counters + kCtrDebugFail, 1ull);
                s_vis[up] = 1;
                if (it_ < p.log_cap) log[it_] = (int32_t)uu;
            }
            __syncwarp();
            const int hp = first_unvisited(s_vis, up + 1, cnt_);
            if (lane == 0) {
                s_m->hpos = hp;
                s_m->head = hp < cnt_ ? s_wl[hp] : kSentinel;
                // the head is the next winner unless a fresh neighbour beats
                // it: start its row towards L2 now
                if (p.pf_spec && hp < cnt_) prefetch_row_l2(p, key_id(s_wl[hp]));
            }
        };
        __syncthreads();
        if (warp == PFW) expand(0, u, 1, 0);
        if (prof) {  // query prologue (filter clear, table, medoid row) -> slot 7
            const long long now_ = clock_after(s_m->ndeg);
            s_m->ph[7] += (unsigned long long)(now_ - s_m->t_ph);
            s_m->t_ph = now_;
        }

        for (;;) {
            ++iters;  // u was expanded (logged, marked) before the last barrier
            const int deg = s_m->ndeg;
            st_probes += deg;
            const bool valid = j < deg;
            // ---- the prefetched row: id, slot, pre-state bit; the code row
            // (L2) in flight while the Bloom test runs
            uint32_t id = 0, ps = 0, cw[MHW];
            uint32_t fl = 0;
            if (STAGE && valid) {
                id = s_nid[j];
                ps = s_nps[tid];
                fl = s_nfl[tid];
                const uint32_t *row = reinterpret_cast<const uint32_t *>(s_code + j * M) + h * MHW;
#pragma unroll
                for (int q = 0; q < MHW; q += 2) {
                    const uint2 v = *reinterpret_cast<const uint2 *>(row + q);
                    cw[q] = v.x;
                    cw[q + 1] = v.y;
                }
            } else if (!STAGE && valid) {
                id = s_nid[j];
                ps = s_nps[tid];
                fl = s_nfl[tid];
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
            const uint32_t mybit = fl & 1u;
            const uint32_t pbit = __shfl_xor_sync(kFull, mybit, 1);
            const uint32_t pps = __shfl_xor_sync(kFull, ps, 1);
            bool fresh = valid && !(mybit && pbit);
            BANG_PF_PHASE(0)  // (phase 1, the zeroing barrier, does not exist here)
            // the fetch-or result tells in-row slot sharing (pf_early: the sets
            // were performed one iteration ahead by the prefetch warps)
            uint32_t old = 0;
            const bool do_atom = fresh && !(h == 1 && pps == ps);
            if (do_atom && !p.pf_early) old = atomicOr(bits + (ps >> 5), 1u << (ps & 31));
            const uint64_t thr = cnt == t ? s_wl[t - 1] : kSentinel;
            uint64_t key = kSentinel;
            bool surv = false;
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
                // (the fetch-or result is consumed only here, after the ADC)
                const bool coll = pass == 0 && do_atom && !mybit &&
                                  (p.pf_early ? (fl & 4u) != 0 : (old & (1u << (ps & 31))) != 0);
                if (lane == 0) {
                    s_m->wmin[warp] = wm;
                    s_m->wcnt[warp] = __popc(sb);
                    s_m->wfresh[warp] = __popc(fb);
                    // this warp's best fresh neighbour may be the next winner
                    if (p.pf_spec && pass == 0 && wm != kSentinel) prefetch_row_l2(p, key_id(wm));
                }
                BANG_PF_PHASE(2)
                const int any_coll = __syncthreads_or(coll);
                BANG_PF_PHASE(3)
                if (any_coll) {
                    // in-row slot sharing: exact replay of the involved probes
                    // by warp 0 from the pre-state bits (replay_row_warp)
                    uint2 *rec = reinterpret_cast<uint2 *>(s_sk);
                    uint8_t *fl2 = reinterpret_cast<uint8_t *>(s_nk);
                    if (h == 0) rec[j].x = ps;
                    else rec[j].y = ps;
                    fl2[2 * j + h] = (uint8_t)((fresh ? 2 : 0) | (mybit ? 4 : 0) | (coll ? 8 : 0));
                    __syncthreads();
                    if (warp == 0) replay_row_warp<RPAD / 32>(rec, fl2, deg, bits, s_fl);
                    __syncthreads();
                    fresh = valid && s_fl[j];
                    continue;  // redo the ADC with the replayed fresh set
                }
                break;
            }
            // ---- eager winner (engine.py:201-205)
            uint64_t best = kSentinel;
            int n = 0, F = 0, woff = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                best = s_m->wmin[w] < best ? s_m->wmin[w] : best;
                if (w < warp) woff += s_m->wcnt[w];
                n += s_m->wcnt[w];
                F += s_m->wfresh[w];
            }
            const uint64_t head = s_m->head;
            const int hpos = s_m->hpos;
            const uint64_t winner = best < head ? best : head;
            const uint32_t wid = winner != kSentinel ? key_id(winner) : 0u;
            st_fresh += F;
            // ---- survivors -> s_nk (warp-aggregated)
            const unsigned sball = __ballot_sync(kFull, surv);
            if (surv) s_nk[woff + __popc(sball & lt)] = key;
            if (pfw) {
                // ---- one hop ahead: the winner's row while warps PFW.. sort + merge
                named_bar_arrive(1, NT);
                const long long c0 = p.profile ? clock64() : 0;
                if (winner != kSentinel) pf_row<NT, MV, PFW>(p, wid, tid, s_code, bits, s_nid, s_nps, s_nfl, s_m);
                if (p.profile && tid == 0) s_m->ph[1] += (unsigned long long)(clock_after(s_nfl[0]) - c0);
            } else {
                named_bar_sync(1, NT);  // all survivors published
                if (p.profile == 2) s_m->t_ph = clock64(); else { BANG_PF_PHASE(4) }
                // ---- kernel 4a: rank sort of the survivors
                for (int q = tc; q < n; q += NC) {
                    const uint64_t k = s_nk[q];
                    int r = 0, i = 0;
                    for (; i + 4 <= n; i += 4)
                        r += (s_nk[i] < k) + (s_nk[i + 1] < k) + (s_nk[i + 2] < k) + (s_nk[i + 3] < k);
                    for (; i < n; ++i) r += s_nk[i] < k;
                    s_sk[r] = k;
                }
                named_bar_sync(2, NC);
                if (p.profile == 2) s_m->t_ph = clock64(); else { BANG_PF_PHASE(5) }
                // ---- kernel 4b: merge + truncate to t (engine.py:210-215)
                if (tc == 0) {
                    int wpos = t;
                    if (winner != kSentinel)
                        wpos = winner != head ? lower_bound_u64(s_wl, cnt, winner)
                                              : hpos + lower_bound_u64(s_sk, n, head);
                    s_m->wpos = wpos;
                }
                uint64_t mv[MAXCH];
                uint8_t mvv[MAXCH];
                int mdst[MAXCH];
#pragma unroll
                for (int c = 0; c < MAXCH; ++c) {
                    const int i = c * NC + tc;
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
                if (tc < n) {
                    sk = s_sk[tc];
                    spos = tc + lower_bound_u64(s_wl, cnt, sk);
                }
                named_bar_sync(2, NC);  // all reads of the old worklist precede the writes
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
                named_bar_sync(2, NC);  // the merged worklist is complete
                if (warp == PFW) {
                    const int wp = s_m->wpos;
                    if (wp < t) expand(wp, wid, min(t, cnt + n), iters);
                }
            }
            cnt = min(t, cnt + n);
            __syncthreads();
            // ---- converge (engine.py:217-236)
            const int wpos = s_m->wpos;
            if (prof) {  // merge + the wait for warp 0's prefetch
                const long long now_ = clock_after(wpos);
                s_m->ph[6] += (unsigned long long)(now_ - s_m->t_ph);
                s_m->t_ph = now_;
            }
            if (wpos >= t) break;
            upos = wpos;
            if (p.debug && tid == 0 && s_wl[upos] != winner) atomicAdd(p.counters + kCtrDebugFail, 1ull);
            u = wid;
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
        BANG_PF_PHASE(7)
    }
#undef BANG_PF_PHASE
    if (p.profile && tc == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) atomicAdd(p.counters + kCtrPhase0 + i, s_m->ph[i]);
    }
    if (tid == 0) {
        atomicAdd(p.counters + kCtrIterations, st_iters);
        atomicAdd(p.counters + kCtrRerank, st_rr);
    }
    if (tc == 0) {
        // probes/fresh were accumulated uniformly by every thread: count once per CTA
        atomicAdd(p.counters + kCtrProbes, st_probes);
        atomicAdd(p.counters + kCtrFresh, st_fresh);
    }
}

}  // namespace bang
