// bang_abi.cu -- the C-ABI of libbang.so (include/bang.h).
//
// Owns device memory for an index handle (codes, codebook, graph, vectors)
// and the per-search workspace, picks the kernel variant for the shapes,
// launches, and implements the visit-log-overflow retry.  Reference seam:
// GraphSearcher.fit/search (engine.py:377-452) -> _search_batch
// (engine.py:108-270) + build_pq_dist_table (pq.py:299-319).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/bang.h"
#include "bang_kernels.cuh"
#include "bang_search_tab.cuh"
#include "bang_search_cta.cuh"
#include "bang_search_pool.cuh"
#include "bang_search_fat.cuh"
#include "bang_search_ctapipe.cuh"
#include "bang_search_pf.cuh"

using namespace bang;

namespace {

thread_local std::string g_err;

bang_status fail(bang_status code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CU(call)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess) {                                                         \
            cudaGetLastError();                                                          \
            return fail(e_ == cudaErrorMemoryAllocation ? BANG_E_OOM : BANG_E_CUDA,      \
                        "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                       \
        }                                                                                \
    } while (0)

template <class T>
struct DevBuf {
    T *p = nullptr;
    size_t n = 0;
    bang_status reserve(size_t want) {
        if (want <= n && p) return BANG_OK;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        size_t bytes = std::max<size_t>(want, 1) * sizeof(T);
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            return fail(BANG_E_OOM, "cudaMalloc(%zu bytes) failed: %s", bytes, cudaGetErrorString(e));
        }
        n = want;
        return BANG_OK;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t align_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

uint64_t host_fnv1a(uint32_t id, uint64_t h) { return fnv1a(id, h); }

}  // namespace

struct bang_index {
    int device = 0;
    int64_t n = 0;
    int32_t m = 0, dim = 0, R = 0, medoid = 0, vec_dtype = 0, placement = 0;
    std::vector<int32_t> sub_sizes, sub_off;
    int32_t uniform_sub = 0;  // sub width if all equal, else 0
    uint8_t *codes = nullptr;
    float *centroids = nullptr;
    int32_t *d_sub_off = nullptr, *d_sub_size = nullptr;
    int32_t *adj = nullptr, *deg = nullptr;
    int32_t *adj_alloc = nullptr;  // allocation base (host-mapped rows carry a header)
    int64_t adj_stride = 0;
    bool row_hdr = false;
    void *vectors = nullptr;
    bool host_graph = false;
    // fat rows (bang_search_fat.cuh): ids + inline neighbour codes, HBM only
    uint8_t *fat = nullptr;
    int64_t fat_stride = 0;
    int32_t fat_code_off = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    int sm_count = 148;
    int max_smem = 227 * 1024;
    int64_t persist_max = 0, window_max = 0;  // L2 persistence limits of the device
    int64_t l2_bytes = 0;                      // L2 capacity of the device
    int64_t smem_per_sm = 0;                   // shared memory per SM
    size_t persist_set = 0;
    // workspace
    DevBuf<float> q, table;
    DevBuf<int32_t> ids, iters, log, overflow, qmap;
    DevBuf<float> dists;
    DevBuf<uint8_t> shortf;
    DevBuf<uint64_t> wall, rr;
    DevBuf<uint32_t> bloom;
    DevBuf<unsigned long long> counters;
    DevBuf<int64_t> offs;
    DevBuf<int32_t> csr;
    DevBuf<uint8_t> skip;
    // last search
    bang_search_stats stats{};
    int64_t last_nq = 0, last_log_cap = 0, log_cap_override = 0;
    bool last_has_table = false, pending = false, last_rerank = false;
    cudaStream_t last_stream = nullptr;
    std::vector<int32_t> last_iters;
    std::vector<int64_t> last_offsets;
    // retry logs (queries whose visit log overflowed the first pass)
    std::vector<int32_t> retry_q;
    int64_t retry_cap = 0;
    DevBuf<int32_t> retry_log;
};

namespace {

struct Plan {
    int variant = kAdcSmemCodebook;
    int npl = 2, sub = 0, mv = 0;
    bool tab_kernel = false;  // search_tab_kernel (smem table + 16-byte code rows)
    bool cta_kernel = false;  // search_cta_kernel (one CTA per query, smem table)
    bool pool_kernel = false; // search_pool_kernel (query pool per CTA, smem codebook)
    bool fat_kernel = false;  // search_fat_kernel (CTA per query over fat rows)
    bool pipe_kernel = false; // search_ctapipe_kernel (next row's loads during the merge)
    bool pf_kernel = false;   // search_pf_kernel (warp 0 prefetches the next row's Bloom bits)
    int pfw = 1;              // search_pf_kernel: prefetch warps
    bool pf_red = false;      // search_pf_kernel: fire-and-forget sets
    bool pf_stage = false;    // search_pf_kernel: next row's code rows staged in smem
    int off_code = 0;
    int off_row = 0;          // CTA kernel: staged host-mapped row (header + ids)
    int off_dup = 0;
    int pool_slots = 0, rr_ctas = 0;
    int nt = 0;               // threads per CTA of the CTA kernel
    int warps = 32, ctas = 148, slots = 0;
    int shared_bytes = 0, per_warp = 0, smem = 0;
    int off_q, off_wl, off_sk, off_nk, off_fid, off_acc, off_alive, off_vis, off_sum, off_tab;
    int sum_words = 0;
    int64_t bloom_stride = 0;
};

template <int NPL, int SUB, int MV>
const void *kernel_ptr() {
    return reinterpret_cast<const void *>(&search_kernel<NPL, SUB, MV>);
}

template <int NPL, int SUB, int MV>
const void *tab_kernel_ptr() {
    return reinterpret_cast<const void *>(&search_tab_kernel<NPL, SUB, MV>);
}

const void *pick_tab_kernel(int npl, int sub, int mv) {
#define BANG_T(N, S, V) \
    if (npl == N && sub == S && mv == V) return tab_kernel_ptr<N, S, V>();
    BANG_T(1, 4, 2) BANG_T(2, 4, 2) BANG_T(4, 4, 2)
    BANG_T(1, 2, 3) BANG_T(2, 2, 3) BANG_T(4, 2, 3)
    BANG_T(1, 0, 2) BANG_T(2, 0, 2) BANG_T(4, 0, 2)
    BANG_T(1, 0, 3) BANG_T(2, 0, 3) BANG_T(4, 0, 3)
#undef BANG_T
    return nullptr;
}

template <int NT, int SUB, int MV>
const void *cta_kernel_ptr(bool hdr) {
    return hdr ? reinterpret_cast<const void *>(&search_cta_kernel<NT, SUB, MV, true>)
               : reinterpret_cast<const void *>(&search_cta_kernel<NT, SUB, MV, false>);
}

const void *pick_cta_kernel(int nt, int sub, int mv, bool hdr = false) {
#define BANG_C(N, S, V) \
    if (nt == N && sub == S && mv == V) return cta_kernel_ptr<N, S, V>(hdr);
    BANG_C(64, 4, 2) BANG_C(128, 4, 2) BANG_C(256, 4, 2)
    BANG_C(64, 2, 3) BANG_C(128, 2, 3) BANG_C(256, 2, 3)
    BANG_C(64, 0, 2) BANG_C(128, 0, 2) BANG_C(256, 0, 2)
    BANG_C(64, 0, 3) BANG_C(128, 0, 3) BANG_C(256, 0, 3)
#undef BANG_C
    return nullptr;
}

template <int N, int S, int V>
const void *pf_kernel_ptr(int pfw, bool stage) {
    if (stage) return pfw == 2 ? reinterpret_cast<const void *>(&search_pf_kernel<N, S, V, 2, true>)
                               : reinterpret_cast<const void *>(&search_pf_kernel<N, S, V, 1, true>);
    return pfw == 2 ? reinterpret_cast<const void *>(&search_pf_kernel<N, S, V, 2, false>)
                    : reinterpret_cast<const void *>(&search_pf_kernel<N, S, V, 1, false>);
}

const void *pick_pf_kernel(int nt, int sub, int mv, int pfw = 1, bool stage = false) {
#define BANG_P(N, S, V) \
    if (nt == N && sub == S && mv == V) return pf_kernel_ptr<N, S, V>(pfw, stage);
    BANG_P(128, 4, 2) BANG_P(256, 4, 2)
    BANG_P(128, 2, 3) BANG_P(256, 2, 3)
    BANG_P(128, 0, 2) BANG_P(256, 0, 2)
    BANG_P(128, 0, 3) BANG_P(256, 0, 3)
#undef BANG_P
    return nullptr;
}

template <int NT, int SUB, int MV>
const void *fat_kernel_ptr() {
    return reinterpret_cast<const void *>(&search_fat_kernel<NT, SUB, MV, MV == 3 ? 4 : 6>);
}

const void *pick_fat_kernel(int nt, int sub, int mv) {
#define BANG_F(N, S, V) \
    if (nt == N && sub == S && mv == V) return fat_kernel_ptr<N, S, V>();
    BANG_F(64, 4, 2) BANG_F(128, 4, 2) BANG_F(64, 2, 3) BANG_F(128, 2, 3)
#undef BANG_F
    return nullptr;
}

template <int NT, int SUB, int MV>
const void *pipe_kernel_ptr() {
    return reinterpret_cast<const void *>(&search_ctapipe_kernel<NT, SUB, MV>);
}

const void *pick_pipe_kernel(int nt, int sub, int mv) {
#define BANG_Q(N, S, V) \
    if (nt == N && sub == S && mv == V) return pipe_kernel_ptr<N, S, V>();
    BANG_Q(64, 4, 2) BANG_Q(128, 4, 2) BANG_Q(256, 4, 2) BANG_Q(64, 2, 3) BANG_Q(128, 2, 3) BANG_Q(256, 2, 3)
    BANG_Q(64, 0, 2) BANG_Q(128, 0, 2) BANG_Q(256, 0, 2) BANG_Q(64, 0, 3) BANG_Q(128, 0, 3) BANG_Q(256, 0, 3)
#undef BANG_Q
    return nullptr;
}

template <int SUB, int MV, int RPAD>
const void *pool_kernel_ptr() {
    return reinterpret_cast<const void *>(&search_pool_kernel<SUB, MV, RPAD>);
}

const void *pick_pool_kernel(int sub, int mv, int rpad) {
#define BANG_P(S, V, P) \
    if (sub == S && mv == V && rpad == P) return pool_kernel_ptr<S, V, P>();
    BANG_P(4, 2, 32) BANG_P(4, 2, 64) BANG_P(2, 3, 32) BANG_P(2, 3, 64)
#undef BANG_P
    return nullptr;
}

// Query-pool plan (search_pool_kernel): CTA-shared codebook + Q slots.
bool plan_pool(bang_index *ix, int64_t nq, int t, int flags, Plan &pl) {
    const int mv = (ix->m % 16 == 0) ? ix->m / 16 : 0;
    const int sub = (ix->uniform_sub == 4 && mv == 2) ? 4 : (ix->uniform_sub == 2 && mv == 3) ? 2 : 0;
    if (!sub || ix->R > 64 || (flags & (BANG_EXACT_DISTANCE | BANG_TABLE_GLOBAL | BANG_TABLE_SMEM |
                                        BANG_CODEBOOK_SMEM | BANG_DEBUG_GENERIC | BANG_WARP_PER_QUERY)))
        return false;
    const int rpad = ix->R <= 32 ? 32 : 64;
    int off = 0;
    auto take = [&](int64_t bytes) { const int o = off; off += (int)align_up(bytes, 16); return o; };
    pl.off_q = take(4LL * ix->dim);
    pl.off_wl = take(8LL * t);
    pl.off_nk = take(8LL * rpad);
    pl.off_sk = take(8LL * rpad);
    pl.off_fid = take(4LL * rpad);
    pl.off_alive = take(rpad);
    pl.off_acc = take(128);  // PoolCtl
    pl.off_vis = take(t);
    pl.off_sum = take(4LL * pl.sum_words);
    pl.off_tab = off;
    pl.per_warp = off;  // bytes per slot
    pl.shared_bytes = (int)align_up((int64_t)256 * ix->dim * 4, 16) + (int)sizeof(PoolCta);
    const int q = (int)std::min<int64_t>(kPoolMaxSlots, (ix->max_smem - pl.shared_bytes) / pl.per_warp);
    if (q < 8) return false;  // too few queries per SM to beat the table kernels
    const void *kp = pick_pool_kernel(sub, mv, rpad);
    if (!kp) return false;
    pl.pool_kernel = true;
    pl.variant = kAdcSmemCodebook;
    pl.sub = sub;
    pl.mv = mv;
    pl.npl = rpad / 32;
    pl.pool_slots = q;
    pl.nt = kPoolThreads;
    pl.warps = kPoolThreads / 32;
    pl.smem = pl.shared_bytes + q * pl.per_warp;
    pl.ctas = (int)std::min<int64_t>(ix->sm_count, std::max<int64_t>(1, ceil_div(nq, q)));
    pl.slots = pl.ctas * q;
    pl.rr_ctas = (int)std::min<int64_t>(4LL * ix->sm_count, std::max<int64_t>(1, ceil_div(nq, 8)));
    return true;
}

const void *pick_kernel(int npl, int sub, int mv) {
#define BANG_K(N, S, V) \
    if (npl == N && sub == S && mv == V) return kernel_ptr<N, S, V>();
    BANG_K(1, 0, 0) BANG_K(2, 0, 0) BANG_K(4, 0, 0)
    BANG_K(1, 4, 2) BANG_K(2, 4, 2) BANG_K(4, 4, 2)
    BANG_K(1, 2, 3) BANG_K(2, 2, 3) BANG_K(4, 2, 3)
    BANG_K(1, 0, 2) BANG_K(2, 0, 2) BANG_K(4, 0, 2)
    BANG_K(1, 0, 3) BANG_K(2, 0, 3) BANG_K(4, 0, 3)
#undef BANG_K
    return nullptr;
}

bang_status make_plan(bang_index *ix, int64_t nq, int t, int64_t z, int flags, Plan &pl) {
    const int Rpad = std::max(32, (int)align_up(ix->R, 32));
    pl.npl = Rpad <= 32 ? 1 : (Rpad <= 64 ? 2 : 4);
    if (ix->R > 128) return fail(BANG_E_PARAM, "degree bound R=%d exceeds 128", ix->R);
    const bool exact = flags & BANG_EXACT_DISTANCE;
    const int64_t cb_bytes = (int64_t)256 * ix->dim * 4;
    // per-warp shared memory: query, worklist keys, sorted/unsorted new
    // keys, fresh ids, partial ADC sums, alive list, visited flags, Bloom
    // summary (one bit per u32 filter word)
    const int rpad = pl.npl * 32;
    pl.bloom_stride = align_up(ceil_div(z, 32), 4);
    pl.sum_words = (int)ceil_div(pl.bloom_stride, 32);
    pl.off_q = 0;
    pl.off_wl = (int)align_up((int64_t)ix->dim * 4, 16);
    pl.off_nk = pl.off_wl + (int)align_up((int64_t)t * 8, 16);
    pl.off_fid = pl.off_nk + (int)align_up((int64_t)rpad * 8, 16);
    pl.off_acc = pl.off_fid + (int)align_up((int64_t)rpad * 4, 16);
    pl.off_alive = pl.off_acc + (int)align_up((int64_t)rpad * 4, 16);
    // the sorted survivors (s_sk, rpad u64) reuse the fid+acc scratch: both
    // are dead once the ADC has produced the survivor keys
    pl.off_sk = pl.off_fid;
    pl.off_vis = pl.off_alive + (int)align_up(rpad, 16);
    pl.off_sum = pl.off_vis + (int)align_up(t, 16);
    pl.per_warp = pl.off_sum + (int)align_up((int64_t)pl.sum_words * 4, 16);
    const int mv = (ix->m % 16 == 0 && ix->m / 16 >= 2 && ix->m / 16 <= 3) ? ix->m / 16 : 0;
    const int64_t tab_bytes = (int64_t)ix->m * 256 * 4;
    const int64_t cb_shared = align_up(cb_bytes + 8LL * ix->m, 16);
    if (exact) {
        pl.variant = kAdcExact;
    } else if (flags & BANG_TABLE_GLOBAL) {
        pl.variant = kAdcGlobalTable;
    } else if (flags & BANG_CODEBOOK_SMEM) {
        if ((ix->max_smem - cb_shared) / pl.per_warp < 1)
            return fail(BANG_E_PARAM, "smem codebook (%lld B) does not fit", (long long)cb_bytes);
        pl.variant = kAdcSmemCodebook;
    } else if (flags & BANG_TABLE_SMEM) {
        if (ix->max_smem / (pl.per_warp + tab_bytes) < 1)
            return fail(BANG_E_PARAM, "a %lld B per-query table does not fit in shared memory", (long long)tab_bytes);
        pl.variant = kAdcSmemTable;
    } else if (ix->max_smem / (pl.per_warp + tab_bytes) >= 4) {
        pl.variant = kAdcSmemTable;   // the paper's layout: per-query table in smem
    } else if ((ix->max_smem - cb_shared) / pl.per_warp >= 8) {
        pl.variant = kAdcSmemCodebook;
    } else {
        pl.variant = kAdcGlobalTable;
    }
    if ((flags & BANG_QUERY_POOL) && !(flags & BANG_NO_POOL)) {
        if (plan_pool(ix, nq, t, flags, pl)) {
            CU(cudaFuncSetAttribute(pick_pool_kernel(pl.sub, pl.mv, pl.npl * 32),
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem));
            return BANG_OK;
        }
        return fail(BANG_E_PARAM, "the query-pool kernel does not support this index/flags (m=%d, sub=%d, R=%d)",
                    ix->m, ix->uniform_sub, ix->R);
    }
    pl.off_tab = pl.per_warp;
    if (pl.variant == kAdcSmemTable) pl.per_warp += (int)tab_bytes;
    if (pl.variant == kAdcSmemCodebook) {
        pl.shared_bytes = (int)cb_shared;
        pl.sub = (ix->uniform_sub == 4 && mv == 2) ? 4 : (ix->uniform_sub == 2 && mv == 3) ? 2 : 0;
        pl.mv = pl.sub ? mv : 0;
    } else if (pl.variant == kAdcSmemTable) {
        pl.shared_bytes = 0;
        pl.sub = (ix->uniform_sub == 4 && mv == 2) ? 4 : (ix->uniform_sub == 2 && mv == 3) ? 2 : 0;
        pl.cta_kernel = mv > 0 && !(flags & (BANG_DEBUG_GENERIC | BANG_WARP_PER_QUERY)) &&
                        t <= 4 * 2 * rpad;
        pl.tab_kernel = mv > 0 && !pl.cta_kernel && !(flags & BANG_DEBUG_GENERIC);
        pl.mv = (pl.sub || pl.tab_kernel || pl.cta_kernel) ? mv : 0;
    } else {
        pl.shared_bytes = 0;
        pl.sub = 0;
        pl.mv = pl.variant == kAdcGlobalTable ? mv : 0;
    }
    if (pl.cta_kernel) {
        // one CTA per query: 2 threads per neighbour slot; CTA-private layout
        pl.nt = 2 * rpad;
        int off = 0;
        auto take = [&](int64_t bytes) { const int o = off; off += (int)align_up(bytes, 16); return o; };
        pl.fat_kernel = ix->fat && !(flags & BANG_NO_FAT) && pl.sub && pick_fat_kernel(pl.nt, pl.sub, pl.mv);
        pl.pipe_kernel = !pl.fat_kernel && (flags & BANG_PIPELINE_ROWS);
        // one-hop-ahead prefetch of the next row by dedicated warps (graph in
        // HBM).  It pays when the next row's loads miss L2 -- codes larger than
        // L2 (C3: 480 MB); with L2-resident codes (C2: 32 MB) the prefetch warps
        // cost more than they hide (-13%).  BANG_PF=1/0 forces it on/off.
        const char *pf = getenv("BANG_PF");
        const bool pf_auto = (int64_t)ix->n * ix->m > (int64_t)ix->l2_bytes;
        // prefetch warps: two halve the per-lane hashing of the next row (C3:
        // 765K vs 739K QPS) while two warps still cover sort + merge at
        // t <= 4*(nt-64); BANG_PF_WARPS=1/2 forces the count
        const char *pfw = getenv("BANG_PF_WARPS");
        pl.pfw = pfw ? (*pfw == '2' ? 2 : 1) : (t <= 4 * (pl.nt - 64) ? 2 : 1);
        pl.pf_kernel = !pl.fat_kernel && !pl.pipe_kernel && !ix->row_hdr &&
                       (pf ? *pf == '1' : pf_auto) &&
                       pl.nt >= 128 && t <= 4 * (pl.nt - 32 * pl.pfw) && pick_pf_kernel(pl.nt, pl.sub, pl.mv, pl.pfw);
        const char *pr = getenv("BANG_PF_RED");
        pl.pf_red = pl.pf_kernel && pr && *pr == '1';
        pl.off_q = take(4LL * ix->dim);
        pl.off_wl = take(8LL * t);
        pl.off_sk = take(8LL * rpad);
        pl.off_nk = take(8LL * rpad);
        pl.off_fid = take(4LL * rpad);
        pl.off_alive = take(rpad);
        pl.off_acc = take(256);  // CtaMisc
        pl.off_vis = take(t);
        // search_pf_kernel clears its filter per query and reads every probe's
        // word: no summary (its 1.5 KB hold the staged code rows instead)
        pl.off_sum = pl.pf_kernel ? 0 : take(4LL * pl.sum_words);
        pl.off_tab = take(tab_bytes);
        if (ix->row_hdr && !pl.fat_kernel && !pl.pipe_kernel) pl.off_row = take(4LL * (rpad + 4));
        if (pl.fat_kernel) {
            pl.off_alive = take(2LL * rpad);            // replay records (flags per probe half)
            pl.off_dup = take(4LL * kDupSlots + rpad);  // slot-sharing table + truly-fresh bytes
        }
        if (pl.pf_kernel) {
            // prefetched slots (u32) + pre-state flags (u8) [+ slot-sharing table]
            pl.off_dup = take(5LL * pl.nt + (pl.pf_red ? 4LL * kDupSlots : 0));
            // the next row's code rows, staged by the prefetch warps when they fit
            const int64_t code_bytes = (int64_t)rpad * 16 * pl.mv;
            const char *st = getenv("BANG_PF_STAGE");
            // (the residency search_pf_kernel's launch bounds target: 4 CTAs of
            // 128 threads at m = 48, 6 at m = 32)
            const int64_t budget = (int64_t)ix->smem_per_sm / std::max(1, (pl.mv == 3 ? 512 : 768) / pl.nt) - 1024;
            pl.pf_stage = !(st && *st == '0') && pl.mv > 0 && off + align_up(code_bytes, 16) <= budget;
            if (pl.pf_stage) pl.off_code = take(code_bytes);
        }
        pl.per_warp = off;  // bytes per CTA
        pl.shared_bytes = 0;
        pl.warps = pl.nt / 32;
        pl.smem = pl.per_warp;
        if (pl.smem > ix->max_smem) return fail(BANG_E_PARAM, "t=%d: %d B of shared memory per query", t, pl.smem);
        const void *kc = pl.fat_kernel    ? pick_fat_kernel(pl.nt, pl.sub, pl.mv)
                         : pl.pipe_kernel ? pick_pipe_kernel(pl.nt, pl.sub, pl.mv)
                         : pl.pf_kernel   ? pick_pf_kernel(pl.nt, pl.sub, pl.mv, pl.pfw, pl.pf_stage)
                                          : pick_cta_kernel(pl.nt, pl.sub, pl.mv, ix->row_hdr);
        if (!kc) return fail(BANG_E_STATE, "no CTA kernel for nt=%d sub=%d mv=%d", pl.nt, pl.sub, pl.mv);
        CU(cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem));
        int per_sm = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kc, pl.nt, pl.smem));
        if (per_sm < 1) return fail(BANG_E_CUDA, "search CTA cannot be resident");
        pl.ctas = (int)std::min<int64_t>((int64_t)ix->sm_count * per_sm, std::max<int64_t>(1, nq));
        pl.slots = pl.ctas;
        return BANG_OK;
    }
    int64_t w = (ix->max_smem - pl.shared_bytes) / pl.per_warp;
    if (w < 1) return fail(BANG_E_PARAM, "t=%d needs %d B of shared memory per query", t, pl.per_warp);
    pl.warps = (int)std::min<int64_t>((pl.tab_kernel ? 256 : kMaxSearchThreads) / 32, w);
    pl.smem = pl.shared_bytes + pl.warps * pl.per_warp;
    const void *kfn = pl.tab_kernel ? pick_tab_kernel(pl.npl, pl.sub, pl.mv) : pick_kernel(pl.npl, pl.sub, pl.mv);
    if (!kfn) return fail(BANG_E_STATE, "no kernel instance for npl=%d sub=%d mv=%d", pl.npl, pl.sub, pl.mv);
    CU(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem));
    int per_sm = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, pl.warps * 32, pl.smem));
    if (per_sm < 1) {
        // registers: shrink the CTA until it fits
        while (pl.warps > 1 && per_sm < 1) {
            pl.warps = pl.warps / 2;
            pl.smem = pl.shared_bytes + pl.warps * pl.per_warp;
            CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, pl.warps * 32, pl.smem));
        }
        if (per_sm < 1) return fail(BANG_E_CUDA, "search kernel cannot be resident");
    }
    pl.ctas = (int)std::min<int64_t>((int64_t)ix->sm_count * per_sm, std::max<int64_t>(1, ceil_div(nq, pl.warps)));
    pl.slots = pl.ctas * pl.warps;
    return BANG_OK;
}

// Enqueue one search pass.  Outputs are indexed by query id; log rows by
// pass index when qmap != nullptr.
bang_status launch_pass(bang_index *ix, const Plan &pl, const float *d_queries, int64_t nq_pass,
                        const int32_t *d_qmap, int k, int t, int64_t z, int flags, int32_t *d_ids,
                        float *d_dists, int32_t *d_iters, uint8_t *d_short, int32_t *d_log,
                        int64_t log_cap, const float *d_table, cudaStream_t st) {
    if (ix->bloom.reserve((size_t)pl.slots * pl.bloom_stride)) return BANG_E_OOM;
    if (ix->rr.reserve((size_t)(pl.pool_kernel ? pl.rr_ctas * 8 : pl.slots) * log_cap)) return BANG_E_OOM;
    SearchParams p{};
    p.codes = ix->codes;
    p.centroids = ix->centroids;
    p.sub_off = ix->d_sub_off;
    p.sub_size = ix->d_sub_size;
    p.table = d_table;
    p.adj = ix->adj;
    p.adj_stride = ix->adj_stride;
    p.row_hdr = ix->row_hdr && pl.cta_kernel && !pl.fat_kernel && !pl.pipe_kernel ? 1 : 0;
    p.off_row = pl.off_row;
    p.deg = ix->deg;
    p.vectors = ix->vectors;
    p.queries = d_queries;
    p.query_map = d_qmap;
    p.nq = nq_pass;
    p.out_ids = d_ids;
    p.out_dists = d_dists;
    p.out_iters = d_iters;
    p.out_short = d_short;
    p.out_wall_ns = ix->wall.p;
    p.visit_log = d_log;
    p.log_cap = log_cap;
    p.rr_scratch = ix->rr.p;
    p.overflow_list = ix->overflow.p;
    p.bloom = ix->bloom.p;
    p.bloom_stride = pl.bloom_stride;
    p.geom.z = (uint64_t)z;
    p.geom.magic = ~0ull / (uint64_t)z;
    p.medoid_p1 = (uint32_t)(host_fnv1a((uint32_t)ix->medoid, kFnvOffset) % (uint64_t)z);
    p.medoid_p2 = (uint32_t)(host_fnv1a((uint32_t)ix->medoid, kFnvOffsetH2) % (uint64_t)z);
    p.counters = ix->counters.p;
    p.m = ix->m;
    p.dim = ix->dim;
    p.R = ix->R;
    p.medoid = ix->medoid;
    p.k = k;
    p.t = t;
    p.vec_dtype = ix->vec_dtype;
    p.adc_variant = pl.variant;
    p.rerank = (flags & BANG_RERANK) ? 1 : 0;
    p.debug = (flags & BANG_DEBUG_CHECKS) ? 1 : 0;
    p.profile = (flags & BANG_PROFILE_PHASES) ? 1 : 0;
    if (p.profile && getenv("BANG_PF_BREAKDOWN")) p.profile = 2;  // pf kernel: slots 4/5 = warp 0's stages
    p.smem_shared_bytes = pl.shared_bytes;
    p.per_warp_bytes = pl.per_warp;
    p.off_q = pl.off_q;
    p.off_wl = pl.off_wl;
    p.off_sk = pl.off_sk;
    p.off_nk = pl.off_nk;
    p.off_fid = pl.off_fid;
    p.off_acc = pl.off_acc;
    p.off_alive = pl.off_alive;
    p.off_vis = pl.off_vis;
    p.off_sum = pl.off_sum;
    p.sum_words = pl.sum_words;
    p.off_tab = pl.off_tab;
    p.pool_slots = pl.pool_slots;
    p.fat = ix->fat;
    p.fat_stride = ix->fat_stride;
    p.fat_code_off = ix->fat_code_off;
    p.off_dup = pl.off_dup;
    {
        const char *bc = getenv("BANG_BLOOM_CLEAR");
        p.bloom_clear = !(bc && *bc == '0');
        const char *pl2 = getenv("BANG_PF_L2");
        p.pf_l2 = pl2 ? atoi(pl2) : 2;
        p.pf_red = pl.pf_red;
        p.pf_stage = pl.pf_stage;
        p.off_code = pl.off_code;
        const char *ps = getenv("BANG_PF_SPEC");
        p.pf_spec = !(ps && *ps == '0');
        const char *ps2 = getenv("BANG_PF_SPEC2");
        p.pf_spec2 = ps2 && *ps2 == '1';  // measured neutral at C3 (795K vs 797K)
        const char *pea = getenv("BANG_PF_EARLY");
        p.pf_early = !pl.pf_red && !(pea && *pea == '0');
        const char *pe = getenv("BANG_PF_EAGER");
        p.pf_eager = pe && *pe == '1';
    }
    // reset the per-pass counters (next-query, stats, overflow) but keep t0
    CU(cudaMemsetAsync(ix->counters.p, 0, sizeof(unsigned long long) * kCtrT0, st));
    CU(cudaMemsetAsync(ix->counters.p + kCtrPhase0, 0, sizeof(unsigned long long) * 8, st));
    if (pl.pool_kernel) {
        void *pargs[] = {&p};
        CU(cudaLaunchKernel(pick_pool_kernel(pl.sub, pl.mv, pl.npl * 32), dim3(pl.ctas), dim3(kPoolThreads), pargs,
                            (size_t)pl.smem, st));
        if (p.rerank)
            rerank_log_kernel<<<pl.rr_ctas, 256, (size_t)8 * ix->dim * sizeof(float), st>>>(p);
        CU(cudaGetLastError());
        return BANG_OK;
    }
    const void *kfn = pl.fat_kernel  ? pick_fat_kernel(pl.nt, pl.sub, pl.mv)
                      : pl.pipe_kernel ? pick_pipe_kernel(pl.nt, pl.sub, pl.mv)
                      : pl.pf_kernel   ? pick_pf_kernel(pl.nt, pl.sub, pl.mv, pl.pfw, pl.pf_stage)
                      : pl.cta_kernel  ? pick_cta_kernel(pl.nt, pl.sub, pl.mv, p.row_hdr != 0)
                      : pl.tab_kernel ? pick_tab_kernel(pl.npl, pl.sub, pl.mv)
                                      : pick_kernel(pl.npl, pl.sub, pl.mv);
    void *args[] = {&p};
    // The per-slot Bloom filters (C2: 888 x 50 KB, C3: 592 x 50 KB) are the
    // search's only re-read random working set; the code/adjacency/vector
    // gathers stream past them.  Mark the filters L2-persisting for this
    // launch (BANG_NO_L2_PERSIST=1 disables) so Bloom words stay L2 hits.
    const char *nopersist = getenv("BANG_NO_L2_PERSIST");
    const size_t bloom_bytes = (size_t)pl.slots * pl.bloom_stride * 4;
    if (ix->persist_max > 0 && !(nopersist && *nopersist == '1')) {
        const size_t win = std::min<size_t>(bloom_bytes, (size_t)ix->persist_max);
        if (ix->persist_set != win) {
            CU(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, win));
            ix->persist_set = win;
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(pl.ctas);
        cfg.blockDim = dim3(pl.warps * 32);
        cfg.dynamicSmemBytes = (size_t)pl.smem;
        cfg.stream = st;
        cudaLaunchAttribute attr{};
        attr.id = cudaLaunchAttributeAccessPolicyWindow;
        attr.val.accessPolicyWindow.base_ptr = ix->bloom.p;
        attr.val.accessPolicyWindow.num_bytes = std::min<size_t>(bloom_bytes, (size_t)ix->window_max);
        attr.val.accessPolicyWindow.hitRatio = 1.0f;
        attr.val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr.val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        CU(cudaLaunchKernelExC(&cfg, kfn, args));
        return BANG_OK;
    }
    CU(cudaLaunchKernel(kfn, dim3(pl.ctas), dim3(pl.warps * 32), args, (size_t)pl.smem, st));
    return BANG_OK;
}

bang_status check_search_args(bang_index *ix, int64_t nq, int k, int t, int64_t z, int flags) {
    if (!ix) return fail(BANG_E_STATE, "GraphSearcher is not fitted (null index)");
    if (nq < 0) return fail(BANG_E_PARAM, "nq must be >= 0");
    if (k < 1 || k > t) return fail(BANG_E_PARAM, "k=%d must be in [1, t=%d]", k, t);
    if (z < 1) return fail(BANG_E_PARAM, "bloom_entries must be >= 1, got %lld", (long long)z);
    if (z >= (1LL << 31)) return fail(BANG_E_PARAM, "bloom_entries must be < 2^31");
    if (!(flags & BANG_EXACT_DISTANCE) && ix->m <= 0)
        return fail(BANG_E_PARAM, "index has no PQ codes; only exact_distance mode is available");
    return BANG_OK;
}

bang_status ensure_outputs(bang_index *ix, int64_t nq, int k, int64_t log_cap) {
    bang_status s;
    if ((s = ix->ids.reserve((size_t)nq * k))) return s;
    if ((s = ix->dists.reserve((size_t)nq * k))) return s;
    if ((s = ix->iters.reserve((size_t)nq))) return s;
    if ((s = ix->shortf.reserve((size_t)nq))) return s;
    if ((s = ix->wall.reserve((size_t)nq))) return s;
    if ((s = ix->overflow.reserve((size_t)nq))) return s;
    if ((s = ix->log.reserve((size_t)nq * log_cap))) return s;
    if ((s = ix->counters.reserve(kCtrCount))) return s;
    return BANG_OK;
}

int64_t default_log_cap(const bang_index *ix, int t) {
    return ix->log_cap_override > 0 ? ix->log_cap_override : std::max<int64_t>(1024, 4LL * t);
}

bang_status enqueue_search(bang_index *ix, const float *d_queries, int64_t nq, int k, int t,
                           int64_t z, int flags, int32_t *d_ids, float *d_dists, int32_t *d_iters,
                           uint8_t *d_short, cudaStream_t st) {
    Plan pl;
    bang_status s = make_plan(ix, nq, t, z, flags, pl);
    if (s) return s;
    const int64_t cap = default_log_cap(ix, t);
    if ((s = ensure_outputs(ix, nq, k, cap))) return s;
    CU(cudaEventRecord(ix->ev[0], st));
    record_t0_kernel<<<1, 1, 0, st>>>(ix->counters.p);
    const float *d_table = nullptr;
    if (pl.variant == kAdcGlobalTable) {
        if ((s = ix->table.reserve((size_t)nq * ix->m * 256))) return s;
        if (nq > 0)
            pq_table_kernel<<<(unsigned)nq, 256, ix->dim * sizeof(float), st>>>(
                ix->centroids, ix->d_sub_off, ix->d_sub_size, ix->m, ix->dim, d_queries, ix->table.p);
        CU(cudaGetLastError());
        d_table = ix->table.p;
    }
    CU(cudaEventRecord(ix->ev[1], st));
    if (nq > 0 &&
        (s = launch_pass(ix, pl, d_queries, nq, nullptr, k, t, z, flags, d_ids, d_dists, d_iters,
                         d_short, ix->log.p, cap, d_table, st)))
        return s;
    CU(cudaEventRecord(ix->ev[2], st));
    ix->stats = bang_search_stats{};
    ix->stats.queries = nq;
    ix->stats.slots = pl.slots;
    ix->stats.warps_per_cta = pl.warps;
    ix->stats.ctas = pl.ctas;
    ix->stats.adc_variant = pl.variant;
    ix->stats.kernel = pl.pool_kernel ? 4 : pl.fat_kernel ? 3 : pl.pipe_kernel ? 5 : pl.pf_kernel ? 6 : pl.cta_kernel ? 2 : pl.tab_kernel ? 1 : 0;
    ix->last_nq = nq;
    ix->last_log_cap = cap;
    ix->last_has_table = d_table != nullptr;
    ix->last_rerank = (flags & BANG_RERANK) != 0;
    ix->last_stream = st;
    ix->pending = true;
    return BANG_OK;
}

// Reads counters after the stream drained; fills stats.
bang_status collect(bang_index *ix, unsigned long long *ctr) {
    CU(cudaStreamSynchronize(ix->last_stream));
    CU(cudaMemcpy(ctr, ix->counters.p, sizeof(unsigned long long) * kCtrCount, cudaMemcpyDeviceToHost));
    float ms_total = 0.f, ms_table = 0.f;
    CU(cudaEventElapsedTime(&ms_table, ix->ev[0], ix->ev[1]));
    CU(cudaEventElapsedTime(&ms_total, ix->ev[1], ix->ev[2]));
    bang_search_stats &S = ix->stats;
    S.iterations = (int64_t)ctr[kCtrIterations];
    S.probes = (int64_t)ctr[kCtrProbes];
    S.fresh = (int64_t)ctr[kCtrFresh];
    S.rerank_cands = (int64_t)ctr[kCtrRerank];
    S.kernel_ms = ms_total;
    S.table_ms = ix->last_has_table ? ms_table : 0.f;
    const int64_t elem = ix->vec_dtype == BANG_VEC_F32 ? 4 : 1;
    // adjacency rows + degree, two Bloom words
    // read per probe and written per admission, code rows of the admitted,
    // re-rank vectors, queries in, results + visit logs out.
    // (fat rows: the code rows of every expanded neighbour arrive with the ids)
    const int64_t code_rows = S.kernel == 3 ? S.probes : S.fresh;
    S.algorithmic_bytes = S.iterations * 8 + S.probes * 4 + S.probes * 8 + S.fresh * 8 +
                          code_rows * ix->m + S.rerank_cands * ix->dim * elem +
                          S.queries * (ix->dim * 4 + 16);
    S.adc_bytes = S.fresh * (ix->m + 12);
    for (int i = 0; i < 8; ++i) S.phase_cycles[i] = (int64_t)ctr[kCtrPhase0 + i];
    ix->pending = false;
    return BANG_OK;
}

}  // namespace

extern "C" {

const char *bang_last_error(void) { return g_err.c_str(); }
const char *bang_version(void) { return "bang-b200 0.1.0 (sm_100a)"; }
int32_t bang_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

bang_status bang_index_create(int32_t device, const uint8_t *codes, int64_t n, int32_t m,
                              const float *centroids, const int32_t *sub_sizes, int32_t dim,
                              const int32_t *adjacency, const int32_t *degrees, int32_t R,
                              int32_t medoid, const void *vectors, int32_t vec_dtype,
                              int32_t graph_placement, bang_index **out) {
    if (!out) return fail(BANG_E_PARAM, "out is NULL");
    *out = nullptr;
    if (n < 1) return fail(BANG_E_PARAM, "graph must contain at least one node");
    if (n >= (1LL << 31)) return fail(BANG_E_PARAM, "node ids must fit in 31 bits");
    if (dim < 1) return fail(BANG_E_PARAM, "dim must be >= 1");
    if (R < 1 || R > 128) return fail(BANG_E_PARAM, "degree bound R=%d must be in [1, 128]", R);
    if (medoid < 0 || medoid >= n) return fail(BANG_E_PARAM, "medoid %d out of range", medoid);
    if (!adjacency || !degrees || !vectors) return fail(BANG_E_PARAM, "adjacency/degrees/vectors required");
    if (vec_dtype < 0 || vec_dtype > 2) return fail(BANG_E_PARAM, "unknown vector dtype %d", vec_dtype);
    if (m < 0 || (m > 0 && (!codes || !centroids || !sub_sizes)))
        return fail(BANG_E_PARAM, "codes/centroids/sub_sizes required when m > 0");
    int ndev = 0;
    CU(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(BANG_E_PARAM, "device %d not available (%d visible)", device, ndev);
    std::vector<int32_t> sz(sub_sizes, sub_sizes + m), off(m);
    int64_t tot = 0;
    for (int s = 0; s < m; ++s) {
        if (sz[s] < 1) return fail(BANG_E_PARAM, "subspace %d has size %d", s, sz[s]);
        off[s] = (int32_t)tot;
        tot += sz[s];
    }
    if (m > 0 && tot != dim) return fail(BANG_E_PARAM, "subspace sizes sum to %lld, expected %d", (long long)tot, dim);
    for (int64_t i = 0; i < n; ++i)
        if (degrees[i] < 0 || degrees[i] > R) return fail(BANG_E_PARAM, "node degree outside [0, degree_bound]");

    CU(cudaSetDevice(device));
    bang_index *ix = new bang_index();
    ix->device = device;
    ix->n = n;
    ix->m = m;
    ix->dim = dim;
    ix->R = R;
    ix->medoid = medoid;
    ix->vec_dtype = vec_dtype;
    ix->placement = graph_placement;
    ix->sub_sizes = sz;
    ix->sub_off = off;
    ix->uniform_sub = 0;
    if (m > 0 && std::all_of(sz.begin(), sz.end(), [&](int v) { return v == sz[0]; })) ix->uniform_sub = sz[0];
    cudaDeviceProp prop;
    auto cleanup_fail = [&](bang_status s) {
        bang_index_destroy(ix);
        return s;
    };
#define CUX(call)                                                                                   \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess) {                                                                    \
            cudaGetLastError();                                                                     \
            return cleanup_fail(fail(e_ == cudaErrorMemoryAllocation ? BANG_E_OOM : BANG_E_CUDA,    \
                                     "%s failed: %s", #call, cudaGetErrorString(e_)));              \
        }                                                                                           \
    } while (0)
    CUX(cudaGetDeviceProperties(&prop, device));
    ix->sm_count = prop.multiProcessorCount;
    ix->max_smem = (int)prop.sharedMemPerBlockOptin;
    ix->persist_max = prop.persistingL2CacheMaxSize;
    ix->l2_bytes = prop.l2CacheSize;
    ix->smem_per_sm = prop.sharedMemPerMultiprocessor;
    ix->window_max = prop.accessPolicyMaxWindowSize;
    CUX(cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking));
    for (auto &e : ix->ev) CUX(cudaEventCreate(&e));
    const size_t elem = vec_dtype == BANG_VEC_F32 ? 4 : 1;
    if (m > 0) {
        CUX(cudaMalloc(&ix->codes, (size_t)n * m));
        CUX(cudaMemcpy(ix->codes, codes, (size_t)n * m, cudaMemcpyHostToDevice));
        CUX(cudaMalloc(&ix->centroids, (size_t)256 * dim * 4));
        CUX(cudaMemcpy(ix->centroids, centroids, (size_t)256 * dim * 4, cudaMemcpyHostToDevice));
        CUX(cudaMalloc(&ix->d_sub_off, sizeof(int32_t) * m));
        CUX(cudaMalloc(&ix->d_sub_size, sizeof(int32_t) * m));
        CUX(cudaMemcpy(ix->d_sub_off, off.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice));
        CUX(cudaMemcpy(ix->d_sub_size, sz.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice));
    }
    const size_t adj_bytes = (size_t)n * R * 4, deg_bytes = (size_t)n * 4, vec_bytes = (size_t)n * dim * elem;
    if (graph_placement == BANG_GRAPH_HOST_MAPPED) {
        // one pinned, mapped host copy read by the kernel over PCIe (the
        // paper's host-resident graph)
        ix->host_graph = true;
        // Rows get a 16-byte header [deg, 0, 0, 0] when R % 4 == 0, so the
        // one-hop-ahead fetch is ONE coalesced read of degree + ids (fewer,
        // larger PCIe read requests than per-thread 4-byte reads)
        ix->row_hdr = R % 4 == 0;
        ix->adj_stride = ix->row_hdr ? R + 4 : R;
        const size_t rows_bytes = (size_t)n * ix->adj_stride * 4;
        CUX(cudaHostAlloc(reinterpret_cast<void **>(&ix->adj_alloc), rows_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
        CUX(cudaHostAlloc(reinterpret_cast<void **>(&ix->deg), deg_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
        CUX(cudaHostAlloc(&ix->vectors, vec_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
        ix->adj = ix->adj_alloc + (ix->row_hdr ? 4 : 0);
        if (ix->row_hdr) {
            for (int64_t i = 0; i < n; ++i) {
                int32_t *row = ix->adj_alloc + i * ix->adj_stride;
                row[0] = degrees[i];
                row[1] = row[2] = row[3] = 0;
                memcpy(row + 4, adjacency + i * R, (size_t)R * 4);
            }
        } else {
            memcpy(ix->adj, adjacency, adj_bytes);
        }
        memcpy(ix->deg, degrees, deg_bytes);
        memcpy(ix->vectors, vectors, vec_bytes);
    } else if (graph_placement == BANG_GRAPH_HBM) {
        ix->adj_stride = R;
        CUX(cudaMalloc(&ix->adj, adj_bytes));
        CUX(cudaMalloc(&ix->deg, deg_bytes));
        CUX(cudaMalloc(&ix->vectors, vec_bytes));
        CUX(cudaMemcpy(ix->adj, adjacency, adj_bytes, cudaMemcpyHostToDevice));
        CUX(cudaMemcpy(ix->deg, degrees, deg_bytes, cudaMemcpyHostToDevice));
        CUX(cudaMemcpy(ix->vectors, vectors, vec_bytes, cudaMemcpyHostToDevice));
        // fat rows for search_fat_kernel: ids + the neighbours' code rows inline
        // (one coalesced read per hop).  Opt-in (BANG_FAT_ROWS=1): measured
        // slower than separate code rows at C2/C3 (profiles/r01/fat_rows.txt)
        const char *fatenv = getenv("BANG_FAT_ROWS");
        if (m > 0 && m % 16 == 0 && m / 16 <= 3 && fatenv && *fatenv == '1') {
            ix->fat_code_off = (int32_t)align_up(4LL * R, 16);
            ix->fat_stride = align_up(ix->fat_code_off + (int64_t)R * m, 16);
            if (cudaMalloc(&ix->fat, (size_t)n * ix->fat_stride) == cudaSuccess) {
                const int64_t blocks = std::min<int64_t>(ceil_div(n * 32, 256), (int64_t)ix->sm_count * 16);
                build_fat_rows_kernel<<<(unsigned)blocks, 256, 0, ix->stream>>>(
                    ix->adj, ix->deg, ix->codes, n, R, m, ix->fat_code_off, ix->fat_stride, ix->fat);
                CUX(cudaGetLastError());
                CUX(cudaStreamSynchronize(ix->stream));
            } else {
                cudaGetLastError();
                ix->fat = nullptr;
            }
        }
    } else {
        return cleanup_fail(fail(BANG_E_PARAM, "unknown graph placement %d", graph_placement));
    }
#undef CUX
    *out = ix;
    return BANG_OK;
}

void bang_index_destroy(bang_index *ix) {
    if (!ix) return;
    cudaSetDevice(ix->device);
    if (ix->stream) cudaStreamSynchronize(ix->stream);
    cudaFree(ix->codes);
    cudaFree(ix->fat);
    cudaFree(ix->centroids);
    cudaFree(ix->d_sub_off);
    cudaFree(ix->d_sub_size);
    if (ix->host_graph) {
        cudaFreeHost(ix->adj_alloc);
        cudaFreeHost(ix->deg);
        cudaFreeHost(ix->vectors);
    } else {
        cudaFree(ix->adj);
        cudaFree(ix->deg);
        cudaFree(ix->vectors);
    }
    ix->q.release();
    ix->table.release();
    ix->ids.release();
    ix->iters.release();
    ix->log.release();
    ix->overflow.release();
    ix->qmap.release();
    ix->dists.release();
    ix->shortf.release();
    ix->wall.release();
    ix->rr.release();
    ix->bloom.release();
    ix->counters.release();
    ix->offs.release();
    ix->csr.release();
    ix->skip.release();
    ix->retry_log.release();
    for (auto e : ix->ev)
        if (e) cudaEventDestroy(e);
    if (ix->stream) cudaStreamDestroy(ix->stream);
    cudaGetLastError();
    delete ix;
}

bang_status bang_index_info(const bang_index *ix, int32_t *device, int64_t *n, int32_t *m, int32_t *dim,
                            int32_t *R) {
    if (!ix) return fail(BANG_E_STATE, "null index");
    if (device) *device = ix->device;
    if (n) *n = ix->n;
    if (m) *m = ix->m;
    if (dim) *dim = ix->dim;
    if (R) *R = ix->R;
    return BANG_OK;
}

bang_status bang_index_device_ptrs(const bang_index *ix, const uint8_t **codes, const float **centroids,
                                   const int32_t **adjacency, const int32_t **degrees, const void **vectors) {
    if (!ix) return fail(BANG_E_STATE, "null index");
    if (codes) *codes = ix->codes;
    if (centroids) *centroids = ix->centroids;
    if (adjacency) *adjacency = ix->adj;
    if (degrees) *degrees = ix->deg;
    if (vectors) *vectors = ix->vectors;
    return BANG_OK;
}

bang_status bang_search_device(bang_index *ix, const float *d_queries, int64_t nq, int32_t k, int32_t t,
                               int64_t bloom_entries, int32_t flags, int32_t *d_ids, float *d_dists,
                               int32_t *d_iterations, uint8_t *d_short, void *stream) {
    bang_status s = check_search_args(ix, nq, k, t, bloom_entries, flags);
    if (s) return s;
    CU(cudaSetDevice(ix->device));
    cudaStream_t st = stream ? reinterpret_cast<cudaStream_t>(stream) : ix->stream;
    return enqueue_search(ix, d_queries, nq, k, t, bloom_entries, flags, d_ids, d_dists, d_iterations,
                          d_short, st);
}

bang_status bang_sync_status(bang_index *ix) {
    if (!ix) return fail(BANG_E_STATE, "null index");
    if (!ix->pending) return BANG_OK;
    CU(cudaSetDevice(ix->device));
    unsigned long long ctr[kCtrCount];
    bang_status s = collect(ix, ctr);
    if (s) return s;
    if (ctr[kCtrDebugFail]) return fail(BANG_E_STATE, "debug check failed: eager candidate disagrees with the worklist head");
    if (ctr[kCtrOverflow] && ix->last_rerank)
        return fail(BANG_E_CAPACITY, "%llu visit logs overflowed the device capacity %lld",
                    (unsigned long long)ctr[kCtrOverflow], (long long)ix->last_log_cap);
    return BANG_OK;
}

bang_status bang_search(bang_index *ix, const float *queries, int64_t nq, int32_t k, int32_t t,
                        int64_t bloom_entries, int32_t flags, int32_t *ids, float *dists,
                        int32_t *iterations, uint8_t *converged, uint8_t *short_, double *wall,
                        int64_t *visit_offsets, int32_t *visit_ids, int64_t visit_cap) {
    bang_status s = check_search_args(ix, nq, k, t, bloom_entries, flags);
    if (s) return s;
    if (nq > 0 && (!queries || !ids || !dists || !iterations)) return fail(BANG_E_PARAM, "NULL output");
    CU(cudaSetDevice(ix->device));
    cudaStream_t st = ix->stream;
    ix->retry_q.clear();
    ix->retry_cap = 0;
    if (nq == 0) {
        ix->stats = bang_search_stats{};
        ix->last_nq = 0;
        ix->last_offsets.assign(1, 0);
        if (visit_offsets) visit_offsets[0] = 0;
        return BANG_OK;
    }
    if ((s = ix->q.reserve((size_t)nq * ix->dim))) return s;
    CU(cudaMemcpyAsync(ix->q.p, queries, sizeof(float) * nq * ix->dim, cudaMemcpyHostToDevice, st));
    if ((s = ensure_outputs(ix, nq, k, default_log_cap(ix, t)))) return s;
    if ((s = enqueue_search(ix, ix->q.p, nq, k, t, bloom_entries, flags, ix->ids.p, ix->dists.p, ix->iters.p,
                            ix->shortf.p, st)))
        return s;
    unsigned long long ctr[kCtrCount];
    if ((s = collect(ix, ctr))) return s;
    if (ctr[kCtrDebugFail])
        return fail(BANG_E_STATE, "debug check failed: eager candidate disagrees with the post-merge worklist head");
    std::vector<int32_t> it(nq);
    CU(cudaMemcpy(it.data(), ix->iters.p, sizeof(int32_t) * nq, cudaMemcpyDeviceToHost));
    const bool want_logs = visit_offsets || visit_ids;
    if (ctr[kCtrOverflow] && (ix->last_rerank || want_logs)) {
        // second pass: only the queries whose visit log overflowed, with a
        // log wide enough for the longest (iterations are deterministic)
        std::vector<int32_t> ov(ctr[kCtrOverflow]);
        CU(cudaMemcpy(ov.data(), ix->overflow.p, sizeof(int32_t) * ov.size(), cudaMemcpyDeviceToHost));
        std::sort(ov.begin(), ov.end());
        int64_t cap2 = 0;
        for (int32_t q : ov) cap2 = std::max<int64_t>(cap2, it[q]);
        Plan pl;
        if ((s = make_plan(ix, (int64_t)ov.size(), t, bloom_entries, flags, pl))) return s;
        if ((s = ix->qmap.reserve(ov.size()))) return s;
        if ((s = ix->retry_log.reserve(ov.size() * (size_t)cap2))) return s;
        CU(cudaMemcpyAsync(ix->qmap.p, ov.data(), sizeof(int32_t) * ov.size(), cudaMemcpyHostToDevice, st));
        const float *d_table = ix->last_has_table ? ix->table.p : nullptr;
        if ((s = launch_pass(ix, pl, ix->q.p, (int64_t)ov.size(), ix->qmap.p, k, t, bloom_entries, flags,
                             ix->ids.p, ix->dists.p, ix->iters.p, ix->shortf.p, ix->retry_log.p, cap2, d_table, st)))
            return s;
        CU(cudaStreamSynchronize(st));
        ix->retry_q = ov;
        ix->retry_cap = cap2;
        ix->stats.retries = (int64_t)ov.size();
    }
    CU(cudaMemcpyAsync(ids, ix->ids.p, sizeof(int32_t) * nq * k, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(dists, ix->dists.p, sizeof(float) * nq * k, cudaMemcpyDeviceToHost, st));
    if (short_) CU(cudaMemcpyAsync(short_, ix->shortf.p, nq, cudaMemcpyDeviceToHost, st));
    std::vector<uint64_t> wns;
    if (wall) {
        wns.resize(nq);
        CU(cudaMemcpyAsync(wns.data(), ix->wall.p, sizeof(uint64_t) * nq, cudaMemcpyDeviceToHost, st));
    }
    CU(cudaStreamSynchronize(st));
    memcpy(iterations, it.data(), sizeof(int32_t) * nq);
    if (converged) memset(converged, 1, nq);  // the loop runs every query to convergence
    if (wall)
        for (int64_t i = 0; i < nq; ++i) wall[i] = (double)wns[i] * 1e-9;
    ix->last_iters = it;
    ix->last_offsets.assign(nq + 1, 0);
    for (int64_t i = 0; i < nq; ++i) ix->last_offsets[i + 1] = ix->last_offsets[i] + it[i];
    if (visit_offsets) memcpy(visit_offsets, ix->last_offsets.data(), sizeof(int64_t) * (nq + 1));
    if (visit_ids) {
        if (ix->last_offsets[nq] > visit_cap)
            return fail(BANG_E_CAPACITY, "visit logs need %lld entries, capacity %lld",
                        (long long)ix->last_offsets[nq], (long long)visit_cap);
        return bang_last_visit_logs(ix, visit_ids, visit_cap);
    }
    return BANG_OK;
}

bang_status bang_last_visit_logs(bang_index *ix, int32_t *visit_ids, int64_t visit_cap) {
    if (!ix) return fail(BANG_E_STATE, "null index");
    const int64_t nq = ix->last_nq;
    if (nq == 0) return BANG_OK;
    if ((int64_t)ix->last_offsets.size() != nq + 1) return fail(BANG_E_STATE, "no completed search on this handle");
    const int64_t total = ix->last_offsets[nq];
    if (total > visit_cap)
        return fail(BANG_E_CAPACITY, "visit logs need %lld entries, capacity %lld", (long long)total,
                    (long long)visit_cap);
    if (total == 0) return BANG_OK;
    CU(cudaSetDevice(ix->device));
    cudaStream_t st = ix->stream;
    bang_status s;
    // compact on the device (first-pass rows + retried rows) -> one D2H copy
    if ((s = ix->offs.reserve((size_t)nq + 1))) return s;
    if ((s = ix->csr.reserve((size_t)total))) return s;
    if ((s = ix->skip.reserve((size_t)nq))) return s;
    std::vector<uint8_t> skip(nq, 0);
    for (int32_t q : ix->retry_q) skip[q] = 1;
    CU(cudaMemcpyAsync(ix->offs.p, ix->last_offsets.data(), sizeof(int64_t) * (nq + 1), cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(ix->skip.p, skip.data(), nq, cudaMemcpyHostToDevice, st));
    compact_logs_kernel<<<(unsigned)ceil_div(nq, 8), 256, 0, st>>>(ix->log.p, ix->last_log_cap, nq, nullptr,
                                                                   ix->offs.p, ix->skip.p, ix->csr.p);
    CU(cudaGetLastError());
    if (!ix->retry_q.empty()) {
        const int64_t nr = (int64_t)ix->retry_q.size();
        compact_logs_kernel<<<(unsigned)ceil_div(nr, 8), 256, 0, st>>>(ix->retry_log.p, ix->retry_cap, nr,
                                                                       ix->qmap.p, ix->offs.p, nullptr, ix->csr.p);
        CU(cudaGetLastError());
    }
    CU(cudaMemcpyAsync(visit_ids, ix->csr.p, sizeof(int32_t) * total, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return BANG_OK;
}

bang_status bang_index_set_log_capacity(bang_index *ix, int64_t capacity) {
    if (!ix) return fail(BANG_E_STATE, "null index");
    if (capacity < 0) return fail(BANG_E_PARAM, "capacity must be >= 0");
    ix->log_cap_override = capacity;
    return BANG_OK;
}

bang_status bang_last_search_stats(const bang_index *ix, bang_search_stats *out) {
    if (!ix || !out) return fail(BANG_E_STATE, "null argument");
    *out = ix->stats;
    return BANG_OK;
}

// ------------------------------------------------------------ per-kernel entries

bang_status bang_pq_table_device(const float *d_centroids, const int32_t *sub_sizes, int32_t m, int32_t dim,
                                 const float *d_queries, int64_t nq, float *d_out, void *stream) {
    if (m < 1 || dim < 1 || !sub_sizes) return fail(BANG_E_PARAM, "bad codebook shape");
    std::vector<int32_t> off(m), sz(sub_sizes, sub_sizes + m);
    int64_t tot = 0;
    for (int s = 0; s < m; ++s) {
        off[s] = (int32_t)tot;
        tot += sz[s];
    }
    if (tot != dim) return fail(BANG_E_PARAM, "subspace sizes sum to %lld, expected %d", (long long)tot, dim);
    if (nq == 0) return BANG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int32_t *d_meta = nullptr;
    CU(cudaMallocAsync(&d_meta, sizeof(int32_t) * 2 * m, st));
    CU(cudaMemcpyAsync(d_meta, off.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(d_meta + m, sz.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, st));
    pq_table_kernel<<<(unsigned)nq, 256, dim * sizeof(float), st>>>(d_centroids, d_meta, d_meta + m, m, dim,
                                                                    d_queries, d_out);
    CU(cudaGetLastError());
    CU(cudaFreeAsync(d_meta, st));
    CU(cudaStreamSynchronize(st));  // the host arrays above are stack-owned
    return BANG_OK;
}

bang_status bang_bloom_filter_device(uint32_t *d_bits, int64_t count, int64_t entries, const int64_t *d_row_offsets,
                                     const uint32_t *d_ids, uint8_t *d_fresh, void *stream) {
    if (entries < 1 || entries >= (1LL << 31)) return fail(BANG_E_PARAM, "bloom_entries must be in [1, 2^31)");
    if (count < 0) return fail(BANG_E_PARAM, "count must be >= 0");
    if (count == 0) return BANG_OK;
    BloomGeom g{(uint64_t)entries, ~0ull / (uint64_t)entries};
    const int64_t words32 = 2 * ceil_div(entries, 64);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    bloom_bank_kernel<<<(unsigned)ceil_div(count, 4), 128, 0, st>>>(d_bits, count, words32, g, d_row_offsets,
                                                                   d_ids, d_fresh);
    CU(cudaGetLastError());
    return BANG_OK;
}

bang_status bang_adc_device(const float *d_table, int32_t m, const uint8_t *d_codes, const int64_t *d_qrows,
                            const uint32_t *d_ids, int64_t n, float *d_dists, uint64_t *d_keys, void *stream) {
    if (m < 1) return fail(BANG_E_PARAM, "m must be >= 1");
    if (n == 0) return BANG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const unsigned grid = (unsigned)ceil_div(n, 256);
    const bool vec_ok = (reinterpret_cast<uintptr_t>(d_codes) % 16) == 0;
    if (vec_ok && m == 32) adc_kernel<2><<<grid, 256, 0, st>>>(d_table, m, d_codes, d_qrows, d_ids, n, d_dists, d_keys);
    else if (vec_ok && m == 48) adc_kernel<3><<<grid, 256, 0, st>>>(d_table, m, d_codes, d_qrows, d_ids, n, d_dists, d_keys);
    else adc_kernel<0><<<grid, 256, 0, st>>>(d_table, m, d_codes, d_qrows, d_ids, n, d_dists, d_keys);
    CU(cudaGetLastError());
    return BANG_OK;
}

bang_status bang_adc_pairs_device(bang_index *ix, const float *d_queries, int64_t nq, const int64_t *d_off,
                                  const uint32_t *d_ids, uint64_t *d_keys, void *stream) {
    if (!ix) return fail(BANG_E_STATE, "null index");
    if (ix->m < 1) return fail(BANG_E_PARAM, "index has no PQ codes");
    if (nq < 0) return fail(BANG_E_PARAM, "nq must be >= 0");
    if (nq == 0) return BANG_OK;
    CU(cudaSetDevice(ix->device));
    cudaStream_t st = stream ? reinterpret_cast<cudaStream_t>(stream) : ix->stream;
    const int mv = (ix->m % 16 == 0) ? ix->m / 16 : 0;
    const int sub = ix->uniform_sub;
    // BANG_ADC_PAIRS=lanes: code rows straight into registers, sums carried
    // across the row's lanes (adc_pairs_lanes_kernel); default: smem-staged rows
    const char *var = std::getenv("BANG_ADC_PAIRS");
    const bool vec = (sub == 4 && mv == 2) || (sub == 2 && mv == 3);
    const bool lanes = vec && var && std::strcmp(var, "lanes") == 0;
    // table + query (+ per-warp double-buffered code-row stages, staged vector path)
    const size_t smem = sizeof(float) * ((size_t)ix->m * 256 + align_up(ix->dim, 4)) +
                        (vec && !lanes ? (size_t)8 * 2 * 32 * ix->m : 0);
    if (smem > (size_t)ix->max_smem) return fail(BANG_E_PARAM, "table of m=%d does not fit in shared memory", ix->m);
    auto launch = [&](const void *fn) -> bang_status {
        CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem));
        const int64_t grid = std::min<int64_t>(nq, (int64_t)ix->sm_count * std::max(1, per_sm));
        int m = ix->m, dim = ix->dim;
        void *args[] = {&ix->centroids, &ix->d_sub_off, &ix->d_sub_size, &m, &dim, &d_queries, &nq,
                        &d_off, &d_ids, &ix->codes, &d_keys};
        CU(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(256), args, smem, st));
        return BANG_OK;
    };
    if (lanes && sub == 4 && mv == 2) return launch(reinterpret_cast<const void *>(&adc_pairs_lanes_kernel<4, 2>));
    if (lanes && sub == 2 && mv == 3) return launch(reinterpret_cast<const void *>(&adc_pairs_lanes_kernel<2, 3>));
    if (sub == 4 && mv == 2) return launch(reinterpret_cast<const void *>(&adc_pairs_kernel<4, 2>));
    if (sub == 2 && mv == 3) return launch(reinterpret_cast<const void *>(&adc_pairs_kernel<2, 3>));
    return launch(reinterpret_cast<const void *>(&adc_pairs_kernel<0, 0>));
}

bang_status bang_sort_rows_device(uint64_t *d_keys, int64_t rows, int32_t width, void *stream) {
    if (width < 0 || width > 6144) return fail(BANG_E_PARAM, "row width %d outside [0, 6144]", width);
    if (rows == 0 || width == 0) return BANG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const size_t smem = sizeof(uint64_t) * width;
    CU(cudaFuncSetAttribute(sort_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    sort_rows_kernel<<<(unsigned)rows, 256, smem, st>>>(d_keys, width);
    CU(cudaGetLastError());
    return BANG_OK;
}

bang_status bang_merge_rows_device(const uint64_t *d_a, const uint8_t *d_a_payload, int64_t rows, int32_t wa,
                                   const uint64_t *d_b, int32_t wb, uint64_t *d_out, uint8_t *d_out_payload,
                                   void *stream) {
    if (wa < 0 || wb < 0) return fail(BANG_E_PARAM, "negative width");
    if (rows == 0 || wa + wb == 0) return BANG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    merge_rows_kernel<<<(unsigned)rows, 128, 0, st>>>(d_a, d_a_payload, wa, d_b, wb, d_out, d_out_payload);
    CU(cudaGetLastError());
    return BANG_OK;
}

bang_status bang_worklist_update_device(uint64_t *d_wl_keys, uint8_t *d_wl_vis, int64_t rows, int32_t t,
                                        const uint64_t *d_new_keys, int32_t w, uint64_t *d_winner, uint8_t *d_done,
                                        void *stream) {
    if (t < 1) return fail(BANG_E_PARAM, "t must be >= 1");
    if (w < 0 || w > 128) return fail(BANG_E_PARAM, "new-key width %d outside [0, 128]", w);
    if (rows == 0) return BANG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int per_warp = (int)(align_up(8LL * t, 16) + 2 * align_up(8LL * w, 16) + align_up(t, 16));
    const int warps = 4;
    const size_t smem = (size_t)per_warp * warps;
    if (smem > 227 * 1024) return fail(BANG_E_PARAM, "t=%d too large for the worklist kernel", t);
    const unsigned grid = (unsigned)ceil_div(rows, warps);
    CU(cudaFuncSetAttribute(worklist_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    worklist_update_kernel<<<grid, warps * 32, smem, st>>>(d_wl_keys, d_wl_vis, rows, t, d_new_keys, w, d_winner,
                                                           d_done);
    CU(cudaGetLastError());
    return BANG_OK;
}

bang_status bang_rerank_device(const void *d_vectors, int32_t vec_dtype, int32_t dim, const float *d_queries,
                               int64_t nq, const int64_t *d_offsets, const int32_t *d_cand_ids, int32_t k,
                               int32_t *d_ids, float *d_dists, uint8_t *d_short, void *stream) {
    if (k < 1 || dim < 1) return fail(BANG_E_PARAM, "k and dim must be >= 1");
    if (nq == 0) return BANG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int64_t total = 0;
    CU(cudaMemcpyAsync(&total, d_offsets + nq, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    uint64_t *scratch = nullptr;
    CU(cudaMallocAsync(&scratch, sizeof(uint64_t) * std::max<int64_t>(total, 1), st));
    const int warps = 4;
    rerank_kernel<<<(unsigned)ceil_div(nq, warps), warps * 32, sizeof(float) * dim * warps, st>>>(
        d_vectors, vec_dtype, dim, d_queries, nq, d_offsets, d_cand_ids, scratch, k, d_ids, d_dists, d_short);
    CU(cudaGetLastError());
    CU(cudaFreeAsync(scratch, st));
    return BANG_OK;
}

bang_status bang_exact_sq_dists_device(const void *d_points, int32_t vec_dtype, int32_t dim, const float *d_queries,
                                       int64_t n, float *d_out, void *stream) {
    if (dim < 1) return fail(BANG_E_PARAM, "dim must be >= 1");
    if (n == 0) return BANG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    exact_dists_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(d_points, vec_dtype, dim, d_queries, n, d_out);
    CU(cudaGetLastError());
    return BANG_OK;
}

}  // extern "C"
