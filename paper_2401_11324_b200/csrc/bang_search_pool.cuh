// bang_search_pool.cuh -- the lockstep query-pool search kernel.
//
// Why a pool: the per-query distance table (kernel 1, m x 256 f32 = 32 KB at
// C2, 48 KB at C3) caps a table-in-smem design at 4-6 queries per SM, and
// each query is a chain of ~100-200 dependent iterations whose every step
// waits on L2/HBM (Bloom words, code rows, adjacency rows, atomics).  Here
// one CTA per SM keeps the CODEBOOK (256 x d f32, shared by all queries) in
// shared memory and runs a pool of Q ~ 24 queries in lockstep:
//
//   phase 1  all Q x R neighbour probes at once: FNV-1a slots, Bloom pre-state
//            words (L2) and the PQ code rows (HBM, 16-byte vectors) in flight
//            together; owner warps expand u (visited flag, visit log, head)
//   phase 2  words first written by a query are zeroed (summary bit set)
//   phase 3  fetch-or atomics of the fresh probes (their return values are
//            only consumed after the ADC, so their latency is hidden), then
//            ADC of every fresh probe from the codebook, 16 subspaces per
//            stage with an exact early exit once the partial sum exceeds the
//            worklist's last key (f32 adds of non-negative terms are monotone)
//   phase 4  (rare) in-row Bloom slot sharing: the owner warp replays the
//            involved probes in adjacency order from registers -- no L2
//            round trips -- and repairs the filter words
//   phase 5  owner warp w (one per slot): eager winner = min(best survivor,
//            first unvisited), the winner's adjacency row is requested, sort
//            survivors, merge + truncate to t, converge; a converged slot is
//            refilled with the next query of the batch at once.
//
// Memory latencies are paid once per pool iteration for Q queries instead of
// once per query iteration.  Table entries are recomputed per lookup in
// pq.py:290-294's op order (bit-identical to kernel 1's table), so results
// equal the reference's bit for bit.  Re-ranking of the
// visit logs runs afterwards in rerank_log_kernel (kernel 5).
#pragma once

#include "bang_kernels.cuh"

namespace bang {

constexpr int kPoolThreads = 768;               // 24 warps; warp w owns slot w
constexpr int kPoolMaxSlots = kPoolThreads / 32;

// Per-slot control block (shared memory; written by the owner warp).
struct PoolCtl {
    long long qi, qid;
    unsigned long long head;  // first unvisited worklist entry after u
    unsigned long long thr;   // survivor bound: wl[t-1] when full, else SENTINEL
    int active, cnt, upos, deg;
    int iters, hpos, coll, nfresh;
    unsigned u;
    int pad[3];
};
static_assert(sizeof(PoolCtl) <= 128, "PoolCtl must fit its 128-byte slot");

// CTA-wide scratch after the codebook (phase profiler: thread 0's cycles)
struct PoolCta {
    unsigned long long ph[8];
    long long t_ph;
    int pad[14];
};
static_assert(sizeof(PoolCta) == 128, "PoolCta is 128 bytes");

template <int SUB, int MV, int RPAD>
__global__ void __launch_bounds__(kPoolThreads, 1) search_pool_kernel(const SearchParams p) {
    constexpr int NT = kPoolThreads;
    constexpr int M = 16 * MV;
    constexpr int IPT = (kPoolMaxSlots * RPAD) / NT;  // probe items per thread
    constexpr int NPL = RPAD / 32;                    // owner-warp keys per lane
    static_assert(IPT >= 1 && IPT * NT == kPoolMaxSlots * RPAD, "item mapping");
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int Q = p.pool_slots, t = p.t, R = p.R;

    float *s_cb = reinterpret_cast<float *>(smem);
    {
        const int n4 = (256 * p.dim) / 4;
        const float4 *src = reinterpret_cast<const float4 *>(p.centroids);
        float4 *dst = reinterpret_cast<float4 *>(s_cb);
        for (int i = tid; i < n4; i += NT) dst[i] = __ldg(src + i);
    }
    PoolCta *s_cta = reinterpret_cast<PoolCta *>(smem + p.smem_shared_bytes - sizeof(PoolCta));
    if (tid == 0) {
        for (int i = 0; i < 8; ++i) s_cta->ph[i] = 0;
        s_cta->t_ph = clock64();
    }
#define BANG_POOL_PHASE(i)                                           \
    if (p.profile && tid == 0) {                                     \
        const long long now_ = clock64();                            \
        s_cta->ph[i] += (unsigned long long)(now_ - s_cta->t_ph);    \
        s_cta->t_ph = now_;                                          \
    }
    auto sbase = [&](int s) { return smem + p.smem_shared_bytes + (size_t)s * p.per_warp_bytes; };
    auto S_q = [&](int s) { return reinterpret_cast<float *>(sbase(s) + p.off_q); };
    auto S_wl = [&](int s) { return reinterpret_cast<uint64_t *>(sbase(s) + p.off_wl); };
    auto S_nk = [&](int s) { return reinterpret_cast<uint64_t *>(sbase(s) + p.off_nk); };
    auto S_sk = [&](int s) { return reinterpret_cast<uint64_t *>(sbase(s) + p.off_sk); };
    auto S_adj = [&](int s) { return reinterpret_cast<uint32_t *>(sbase(s) + p.off_fid); };
    auto S_fl = [&](int s) { return sbase(s) + p.off_alive; };
    auto S_ctl = [&](int s) { return reinterpret_cast<PoolCtl *>(sbase(s) + p.off_acc); };
    auto S_vis = [&](int s) { return sbase(s) + p.off_vis; };
    auto S_sum = [&](int s) { return reinterpret_cast<uint32_t *>(sbase(s) + p.off_sum); };
    auto S_bits = [&](int s) { return p.bloom + ((int64_t)blockIdx.x * Q + s) * p.bloom_stride; };

    unsigned long long st_iters = 0, st_probes = 0, st_fresh = 0;

    // ---- owner warp: take the next query of the batch into slot s (or retire it)
    auto slot_start = [&](int s) {
        PoolCtl *c = S_ctl(s);
        long long qi = 0;
        if (lane == 0) qi = (long long)atomicAdd(p.counters + kCtrNextQuery, 1ull);
        qi = __shfl_sync(kFull, qi, 0);
        if (qi >= p.nq) {
            if (lane == 0) c->active = 0;
            __syncwarp();
            return;
        }
        const long long qid = p.query_map ? (long long)p.query_map[qi] : qi;
        float *q = S_q(s);
        uint32_t *sum = S_sum(s);
        uint8_t *vis = S_vis(s);
        uint32_t *bits = S_bits(s);
        for (int i = lane; i < p.dim; i += 32) q[i] = __ldg(p.queries + qid * p.dim + i);
        for (int i = lane; i < p.sum_words; i += 32) sum[i] = 0u;
        for (int i = lane; i < t; i += 32) vis[i] = 0;
        __syncwarp();
        if (lane == 0) {  // the medoid in the filter (engine.py:127-128)
            const uint32_t w1 = p.medoid_p1 >> 5, w2 = p.medoid_p2 >> 5;
            const uint32_t b1 = 1u << (p.medoid_p1 & 31), b2 = 1u << (p.medoid_p2 & 31);
            if (w1 == w2) {
                __stcg(bits + w1, b1 | b2);
            } else {
                __stcg(bits + w1, b1);
                __stcg(bits + w2, b2);
            }
            sum[w1 >> 5] |= 1u << (w1 & 31);
            sum[w2 >> 5] |= 1u << (w2 & 31);
            // worklist = [key(ADC(medoid), medoid)] (engine.py:118-125)
            const float d0 = adc_codebook<SUB, MV>(s_cb, q, nullptr, nullptr, M, p.codes + (int64_t)p.medoid * M);
            S_wl(s)[0] = pack_key(d0, (uint32_t)p.medoid);
            c->qi = qi;
            c->qid = qid;
            c->active = 1;
            c->cnt = 1;
            c->upos = 0;
            c->iters = 0;
            c->u = (uint32_t)p.medoid;
            c->deg = p.deg[p.medoid];
        }
        uint32_t *adj = S_adj(s);
        for (int j = lane; j < RPAD; j += 32) adj[j] = j < R ? (uint32_t)p.adj[(int64_t)p.medoid * p.adj_stride + j] : 0u;
        __syncwarp();
    };

    // ---- owner warp: outputs of a converged query (engine.py:244-269)
    auto slot_finish = [&](int s) {
        PoolCtl *c = S_ctl(s);
        const long long qid = c->qid;
        const int iters = c->iters;
        st_iters += iters;
        if (lane == 0) {
            p.out_iters[qid] = iters;
            p.out_wall_ns[qid] = globaltimer_ns() - p.counters[kCtrT0];
            if (p.log_cap < iters) {  // truncated visit log: the host re-runs this query
                const unsigned long long at = atomicAdd(p.counters + kCtrOverflow, 1ull);
                p.overflow_list[at] = (int32_t)qid;
            }
        }
        if (!p.rerank) {  // wl[0:k] (engine.py:263-265); re-rank is rerank_log_kernel
            const uint64_t *wl = S_wl(s);
            const int cnt = c->cnt;
            for (int i = lane; i < p.k; i += 32) {
                if (i < cnt) {
                    p.out_ids[qid * p.k + i] = (int32_t)key_id(wl[i]);
                    p.out_dists[qid * p.k + i] = key_dist(wl[i]);
                } else {
                    p.out_ids[qid * p.k + i] = -1;
                    p.out_dists[qid * p.k + i] = __int_as_float(0x7f800000);
                }
            }
            if (lane == 0) p.out_short[qid] = cnt < p.k;
        }
        __syncwarp();
    };

    __syncthreads();  // codebook resident
    if (warp < Q) slot_start(warp);

    for (;;) {
        if (!__syncthreads_or(warp < Q && lane == 0 && S_ctl(warp)->active)) break;
        BANG_POOL_PHASE(7)  // loop-top barrier (waits for the slowest owner warp)

        // ================= phase 1: probes (pre-state) + code rows in flight
        uint32_t ps1[IPT], ps2[IPT], w1[IPT], w2[IPT], o1[IPT], o2[IPT], nid[IPT];
        bool valid[IPT], fresh[IPT], in1[IPT], in2[IPT];
        uint4 cw[IPT][MV];
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            const int item = tid + k * NT, s = item / RPAD, j = item % RPAD;
            valid[k] = false;
            ps1[k] = ps2[k] = w1[k] = w2[k] = o1[k] = o2[k] = nid[k] = 0;
            in1[k] = in2[k] = true;
            if (s < Q) {
                const PoolCtl *c = S_ctl(s);
                valid[k] = c->active && j < c->deg;
            }
            if (valid[k]) {
                const uint32_t id = S_adj(s)[j];
                nid[k] = id;
                const uint4 *row = reinterpret_cast<const uint4 *>(p.codes + (int64_t)id * M);
#pragma unroll
                for (int v = 0; v < MV; ++v) cw[k][v] = __ldg(row + v);
                ps1[k] = mod_z(fnv1a(id, kFnvOffset), p.geom);
                ps2[k] = mod_z(fnv1a(id, kFnvOffsetH2), p.geom);
                const uint32_t *sum = S_sum(s);
                const uint32_t *bits = S_bits(s);
                in1[k] = sum_get(sum, ps1[k] >> 5);
                in2[k] = sum_get(sum, ps2[k] >> 5);
                if (in1[k]) w1[k] = __ldcg(bits + (ps1[k] >> 5));
                if (in2[k]) w2[k] = __ldcg(bits + (ps2[k] >> 5));
            }
        }
        // owner warps expand u (engine.py:163-178) while the loads fly
        if (warp < Q) {
            PoolCtl *c = S_ctl(warp);
            if (c->active) {
                uint8_t *vis = S_vis(warp);
                const int upos = c->upos, cnt = c->cnt, iters = c->iters;
                if (lane == 0) {
                    if (p.debug && key_id(S_wl(warp)[upos]) != c->u) atomicAdd(p.counters + kCtrDebugFail, 1ull);
                    vis[upos] = 1;
                    if (iters < p.log_cap) p.visit_log[(p.query_map ? c->qi : c->qid) * p.log_cap + iters] = (int32_t)c->u;
                }
                __syncwarp();
                const int hp = first_unvisited(vis, upos + 1, cnt);
                if (lane == 0) {
                    const uint64_t *wl = S_wl(warp);
                    c->hpos = hp;
                    c->head = hp < cnt ? wl[hp] : kSentinel;
                    c->thr = cnt == t ? wl[t - 1] : kSentinel;
                    c->iters = iters + 1;
                    c->coll = 0;
                    c->nfresh = 0;
                }
                st_probes += c->deg;
            }
        }
        BANG_POOL_PHASE(0)  // issue + owner expand
#pragma unroll
        for (int k = 0; k < IPT; ++k)
            fresh[k] = valid[k] && !(((w1[k] >> (ps1[k] & 31)) & 1u) && ((w2[k] >> (ps2[k] & 31)) & 1u));
        if (p.profile) asm volatile("" ::"r"((int)fresh[0]));
        BANG_POOL_PHASE(1)  // Bloom word loads landed (thread 0)
        __syncthreads();  // every summary read and pre-state load precedes the writes below
        BANG_POOL_PHASE(2)  // barrier: slowest load in the CTA

        // ================= phase 2: words first written by this query
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            if (fresh[k] && (!in1[k] || !in2[k])) {
                const int s = (tid + k * NT) / RPAD;
                uint32_t *sum = S_sum(s);
                uint32_t *bits = S_bits(s);
                if (!in1[k]) {
                    __stcg(bits + (ps1[k] >> 5), 0u);
                    sum_set(sum, ps1[k] >> 5);
                }
                if (!in2[k]) {
                    __stcg(bits + (ps2[k] >> 5), 0u);
                    sum_set(sum, ps2[k] >> 5);
                }
            }
        }
        __syncthreads();  // zeroing stores (any thread) before any atomic
        BANG_POOL_PHASE(3)

        // ================= phase 3: atomics in flight, ADC from the codebook
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            if (fresh[k]) {
                uint32_t *bits = S_bits((tid + k * NT) / RPAD);
                o1[k] = atomicOr(bits + (ps1[k] >> 5), 1u << (ps1[k] & 31));
                if (ps2[k] != ps1[k]) o2[k] = atomicOr(bits + (ps2[k] >> 5), 1u << (ps2[k] & 31));
            }
        }
        bool coll = false;
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            const int item = tid + k * NT, s = item / RPAD, j = item % RPAD;
            if (s >= Q) continue;
            uint64_t key = kSentinel;
            if (fresh[k]) {
                const PoolCtl *c = S_ctl(s);
                const uint64_t thr = c->thr;
                const float thr_d = thr == kSentinel ? __int_as_float(0x7f800000) : key_dist(thr);
                const float *q = S_q(s);
                float acc = 0.0f;
                bool alive = true;
#pragma unroll
                for (int v = 0; v < MV; ++v) {
                    if (alive) {
                        acc = adc_cb_stage16<SUB>(acc, s_cb, q, 16 * v, cw[k][v]);
                        if (v < MV - 1 && acc > thr_d) alive = false;  // exact early exit
                    }
                }
                if (alive) {
                    key = pack_key(acc, nid[k]);
                    if (!(key < thr)) key = kSentinel;  // ranks >= t are truncated (engine.py:213)
                }
            }
            S_nk(s)[j] = key;
            // warp-aggregated fresh count (the 32 items of one k share a slot)
            const unsigned fb = __ballot_sync(kFull, fresh[k]);
            if (lane == 0 && fb) atomicAdd(&S_ctl(s)->nfresh, __popc(fb));
            if (fresh[k]) {
                const uint32_t b1 = 1u << (ps1[k] & 31), b2 = 1u << (ps2[k] & 31);
                const bool c1 = (o1[k] & b1) && !(w1[k] & b1);
                const bool c2 = ps2[k] != ps1[k] && (o2[k] & b2) && !(w2[k] & b2);
                if (c1 || c2) {
                    coll = true;
                    S_ctl(s)->coll = 1;
                }
            }
        }
        BANG_POOL_PHASE(4)  // atomics + ADC (thread 0's items)
        const int any_coll = __syncthreads_or(coll);
        BANG_POOL_PHASE(5)  // barrier: slowest ADC in the CTA
        if (any_coll) {
            // ============= phase 4 (rare): in-row slot sharing, exact replay
            // probe records of the rows with a collision -> smem scratch
#pragma unroll
            for (int k = 0; k < IPT; ++k) {
                const int item = tid + k * NT, s = item / RPAD, j = item % RPAD;
                if (s < Q && S_ctl(s)->coll) {
                    reinterpret_cast<uint2 *>(S_sk(s))[j] = make_uint2(ps1[k], ps2[k]);
                    const uint32_t b1 = 1u << (ps1[k] & 31), b2 = 1u << (ps2[k] & 31);
                    const bool c1 = fresh[k] && (o1[k] & b1) && !(w1[k] & b1);
                    const bool c2 = fresh[k] && ps2[k] != ps1[k] && (o2[k] & b2) && !(w2[k] & b2);
                    S_fl(s)[j] = (uint8_t)((fresh[k] ? 1 : 0) | ((w1[k] & b1) ? 2 : 0) | ((w2[k] & b2) ? 4 : 0) |
                                           ((c1 || c2) ? 8 : 0));
                }
            }
            __syncthreads();
            if (warp < Q && S_ctl(warp)->coll) {
                const int s = warp;
                const uint2 *pp = reinterpret_cast<const uint2 *>(S_sk(s));
                const uint8_t *fl = S_fl(s);
                const int deg = S_ctl(s)->deg;
                uint32_t a[NPL], b[NPL], f[NPL];
#pragma unroll
                for (int r = 0; r < NPL; ++r) {
                    const int j = lane + 32 * r;
                    const uint2 v = j < deg ? pp[j] : make_uint2(0xFFFFFFFFu, 0xFFFFFFFEu);
                    a[r] = v.x;
                    b[r] = v.y;
                    f[r] = j < deg ? fl[j] : 0u;
                }
                // involved probes: presumed fresh and sharing a slot with a colliding probe
                bool inv[NPL];
#pragma unroll
                for (int r = 0; r < NPL; ++r) inv[r] = (f[r] & 8u) != 0;
#pragma unroll
                for (int rc = 0; rc < NPL; ++rc) {
                    unsigned cm = __ballot_sync(kFull, (f[rc] & 8u) != 0);
                    while (cm) {
                        const int src = __ffs(cm) - 1;
                        cm &= cm - 1;
                        const uint32_t pa = __shfl_sync(kFull, a[rc], src), pb = __shfl_sync(kFull, b[rc], src);
#pragma unroll
                        for (int r = 0; r < NPL; ++r)
                            inv[r] = inv[r] || ((f[r] & 1u) && (a[r] == pa || a[r] == pb || b[r] == pa || b[r] == pb));
                    }
                }
                // replay the involved probes in adjacency order (bloom.py:110-122);
                // tf = involved probes found truly fresh so far (only involved
                // probes can share a slot, so they alone make up the row's set)
                bool tf[NPL], drop[NPL];
#pragma unroll
                for (int r = 0; r < NPL; ++r) tf[r] = drop[r] = false;
                auto in_set = [&](uint32_t pos) {
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
                        const uint32_t fj = __shfl_sync(kFull, f[r], src);
                        const bool h1 = (fj & 2u) || in_set(pa);
                        const bool h2 = (fj & 4u) || in_set(pb);
                        if (lane == src) {
                            if (!(h1 && h2)) tf[r] = true;
                            else drop[r] = true;  // an earlier probe of this row set its bits
                        }
                    }
                }
                // repair: a dropped probe's bits that neither the pre-state nor a
                // truly fresh probe holds go back to 0 (its fetch-or completed
                // before the barrier above)
                uint32_t *bits = S_bits(s);
                int ndrop = 0;
#pragma unroll
                for (int r = 0; r < NPL; ++r) {
                    unsigned dm = __ballot_sync(kFull, drop[r]);
                    ndrop += __popc(dm);
                    while (dm) {
                        const int src = __ffs(dm) - 1;
                        dm &= dm - 1;
                        const uint32_t pa = __shfl_sync(kFull, a[r], src), pb = __shfl_sync(kFull, b[r], src);
                        const uint32_t fj = __shfl_sync(kFull, f[r], src);
                        const bool keep_a = (fj & 2u) || in_set(pa);
                        const bool keep_b = pb == pa || (fj & 4u) || in_set(pb);
                        if (lane == 0) {
                            if (!keep_a) atomicAnd(bits + (pa >> 5), ~(1u << (pa & 31)));
                            if (!keep_b) atomicAnd(bits + (pb >> 5), ~(1u << (pb & 31)));
                            S_nk(s)[src + 32 * r] = kSentinel;
                        }
                    }
                }
                if (lane == 0) S_ctl(s)->nfresh -= ndrop;
                __syncwarp();
            }
            __syncthreads();
        }

        // ================= phase 5: owner warps -- eager winner, sort, merge, converge
        if (warp < Q) {
            const int s = warp;
            PoolCtl *c = S_ctl(s);
            if (c->active) {
                uint64_t *nk = S_nk(s);
                uint64_t *sk = S_sk(s);
                uint64_t *wl = S_wl(s);
                uint8_t *vis = S_vis(s);
                // survivors (keys < thr) -> compact, warp min
                uint64_t kv[NPL];
                uint64_t mn = kSentinel;
#pragma unroll
                for (int r = 0; r < NPL; ++r) {
                    kv[r] = nk[lane + 32 * r];
                    mn = kv[r] < mn ? kv[r] : mn;
                }
                mn = warp_min_u64(mn);
                const uint64_t head = c->head;
                const uint64_t winner = mn < head ? mn : head;
                // ---- one-hop-ahead fetch of the winner's adjacency row
                uint32_t na[NPL];
                int ndeg = 0;
                if (winner != kSentinel) {
                    const uint32_t w = key_id(winner);
                    ndeg = p.deg[w];
#pragma unroll
                    for (int r = 0; r < NPL; ++r) {
                        const int j = lane + 32 * r;
                        na[r] = j < R ? (uint32_t)p.adj[(int64_t)w * p.adj_stride + j] : 0u;
                    }
                }
                __syncwarp();
                int n = 0;
#pragma unroll
                for (int r = 0; r < NPL; ++r) {
                    const bool keep = kv[r] != kSentinel;
                    const unsigned bal = __ballot_sync(kFull, keep);
                    if (keep) nk[n + __popc(bal & lt)] = kv[r];
                    n += __popc(bal);
                }
                __syncwarp();
                st_fresh += c->nfresh;
                // ---- kernel 4: sort survivors, merge + truncate (engine.py:210-215)
                sort_keys(nk, n, sk);
                const int hpos = c->hpos;
                int first = 0;
                const int cnt = merge_sorted(wl, vis, c->cnt, t, sk, n, &first);
                int wpos = t;
                if (winner != kSentinel) wpos = mn < head ? first : hpos + lower_bound_u64(sk, n, head);
                __syncwarp();
                if (lane == 0) c->cnt = cnt;
                __syncwarp();
                if (wpos >= t) {  // converged (engine.py:217)
                    slot_finish(s);
                    slot_start(s);
                } else {
                    if (p.debug && lane == 0 && wl[wpos] != winner) atomicAdd(p.counters + kCtrDebugFail, 1ull);
                    uint32_t *adj = S_adj(s);
#pragma unroll
                    for (int r = 0; r < NPL; ++r) adj[lane + 32 * r] = na[r];
                    if (lane == 0) {
                        c->upos = wpos;
                        c->u = key_id(winner);
                        c->deg = ndeg;
                    }
                    __syncwarp();
                }
            }
        }
        BANG_POOL_PHASE(6)  // rare replay + owner phase (slot 0)
    }
#undef BANG_POOL_PHASE
    if (p.profile && tid == 0)
        for (int i = 0; i < 8; ++i) atomicAdd(p.counters + kCtrPhase0 + i, s_cta->ph[i]);
    if (lane == 0) {
        atomicAdd(p.counters + kCtrIterations, st_iters);
        atomicAdd(p.counters + kCtrProbes, st_probes);
        atomicAdd(p.counters + kCtrFresh, st_fresh);
    }
}

// Kernel 5 after the pool search: exact distances of each visit log, top-k
// (engine.py:244-262) -- the same arithmetic as the fused kernels' epilogue.
// One warp per query; queries whose log overflowed are left to the retry.
__global__ void __launch_bounds__(256) rerank_log_kernel(const SearchParams p) {
    extern __shared__ float s_qv[];
    const int warp = threadIdx.x >> 5, lane = (int)lane_id();
    const int nw = blockDim.x >> 5;
    float *q = s_qv + (size_t)warp * p.dim;
    const int64_t gw = (int64_t)blockIdx.x * nw + warp, stride = (int64_t)gridDim.x * nw;
    uint64_t *rr = p.rr_scratch + gw * p.log_cap;
    unsigned long long st_rr = 0;
    for (int64_t qi = gw; qi < p.nq; qi += stride) {
        const int64_t qid = p.query_map ? (int64_t)p.query_map[qi] : qi;
        const int iters = p.out_iters[qid];
        if (iters > p.log_cap) continue;
        for (int j = lane; j < p.dim; j += 32) q[j] = __ldg(p.queries + qid * p.dim + j);
        __syncwarp();
        const int32_t *log = p.visit_log + (p.query_map ? qi : qid) * p.log_cap;
        for (int i = lane; i < iters; i += 32) {
            const uint32_t node = (uint32_t)__ldg(log + i);
            rr[i] = pack_key(exact_sq_dist(p.vectors, p.vec_dtype, p.dim, node, q), node);
        }
        st_rr += iters;
        __threadfence_block();
        __syncwarp();
        warp_topk_write(rr, iters, p.k, p.out_ids + qid * p.k, p.out_dists + qid * p.k);
        if (lane == 0) p.out_short[qid] = iters < p.k;
        __syncwarp();
    }
    if (lane == 0) atomicAdd(p.counters + kCtrRerank, st_rr);
}

}  // namespace bang
