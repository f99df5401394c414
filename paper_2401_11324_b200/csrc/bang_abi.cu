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
#include <map>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "../../include/bang.h"
#include "bang_kernels.cuh"
#include "bang_pick.h"
#include "bang_standalone.cuh"

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

}  // namespace

namespace bang {
// the thread-local message of bang_last_error() for the other translation units
bang_status set_error_msg(bang_status code, const char *msg) {
    g_err = msg;
    return code;
}
}  // namespace bang

namespace {

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
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    bang_options opts{};
    int32_t code_stride = 0;  // bytes between code rows (m, or 64 for m = 48)
    int32_t k_last = 0;       // k of the last search (stats)
    bool persist_user = false;
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
    unsigned long long *h_ctr = nullptr;  // pinned copy of the counters (one-batch readback)
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
    // degree | in-row Bloom slot sharing << 31 at z = row_share_z (bloom_direct)
    DevBuf<int32_t> row_share;
    int64_t row_share_z = 0;
};

namespace {

// stats.kernel ids (bang.h)
enum KernelId { kKGeneric = 0, kKCta = 2, kKSplit = 8 };

struct Plan {
    int variant = kAdcSmemCodebook;
    int kernel = kKGeneric;
    int npl = 2, sub = 0, mv = 0;
    int off_code = 0;
    int off_hrow = 0;         // split kernel: staged head row ids
    int off_row = 0;          // CTA kernel: staged host-mapped row (header + ids)
    int off_dup = 0;
    int nt = 0;               // threads per CTA of the CTA kernels
    int warps = 32, ctas = 148, slots = 0;
    int shared_bytes = 0, per_warp = 0, smem = 0;
    int off_q, off_wl, off_sk, off_nk, off_fid, off_acc, off_alive, off_vis, off_sum, off_tab;
    int sum_words = 0;
    int64_t bloom_stride = 0;
    const void *fn = nullptr;  // the kernel to launch
};

// Kernel + shared-memory layout for one search pass.  Kernel choice
// (bang_options.kernel, BANG_KERNEL_AUTO by default):
//   exact distances, the HBM table, the shared codebook or BANG_KERNEL_WARP
//     -> search_kernel (one warp per query, every ADC data flow);
//   16-byte code rows (m = 32 or 48) with the per-query smem table
//     -> search_split_kernel for an HBM graph and t <= 256 (row warps and
//        list warps overlap a hop's memory phase with the previous hop's
//        merge; measured 1.37x search_cta_kernel at C2 and C3), else
//        search_cta_kernel (host-mapped graphs, longer worklists);
//   anything else -> search_kernel.
bang_status make_plan(bang_index *ix, int64_t nq, int t, int64_t z, int flags, Plan &pl) {
    const bang_options &o = ix->opts;
    const int Rpad = std::max(32, (int)align_up(ix->R, 32));
    pl.npl = Rpad <= 32 ? 1 : (Rpad <= 64 ? 2 : 4);
    if (ix->R > 128) return fail(BANG_E_PARAM, "degree bound R=%d exceeds 128", ix->R);
    const bool exact = flags & BANG_EXACT_DISTANCE;
    const int64_t cb_bytes = (int64_t)256 * ix->dim * 4;
    const int rpad = pl.npl * 32;
    pl.bloom_stride = align_up(ceil_div(z, 32), 4);
    pl.sum_words = (int)ceil_div(pl.bloom_stride, 32);
    const int mv = (ix->m % 16 == 0 && ix->m / 16 >= 2 && ix->m / 16 <= 3) ? ix->m / 16 : 0;
    const int vsub = (ix->uniform_sub == 4 && mv == 2) ? 4 : (ix->uniform_sub == 2 && mv == 3) ? 2 : 0;
    const int64_t tab_bytes = (int64_t)ix->m * 256 * 4;
    const bool forced_generic = exact || (flags & (BANG_TABLE_GLOBAL | BANG_CODEBOOK_SMEM)) ||
                                o.kernel == BANG_KERNEL_WARP;
    if ((o.kernel == BANG_KERNEL_CTA || o.kernel == BANG_KERNEL_SPLIT) && (forced_generic || mv == 0))
        return fail(BANG_E_PARAM, "the CTA kernels need m = 32 or 48 with the smem table (m=%d, flags=%d)", ix->m,
                    flags);
    // ---- one CTA per query, row warps + list warps (search_split_kernel)
    const bool split_ok = t <= 256;
    if (o.kernel == BANG_KERNEL_SPLIT && !split_ok)
        return fail(BANG_E_PARAM, "search_split_kernel needs t <= 256 (t=%d)", t);
    // AUTO: split for HBM graphs; host-mapped rows go to search_cta_kernel,
    // whose warp-0 16-byte row copies make fewer PCIe read requests (C4r:
    // 259 K vs 224 K QPS, profiles/r02/bench_C4r_*.json)
    const bool split_auto = o.kernel == BANG_KERNEL_AUTO && !ix->host_graph;
    if (!forced_generic && mv > 0 && split_ok && (o.kernel == BANG_KERNEL_SPLIT || split_auto)) {
        const int spl = rpad <= 64 ? 1 : 2;
        const int srpad = 64 * spl;
        pl.variant = kAdcSmemTable;
        pl.sub = vsub;
        pl.mv = mv;
        pl.nt = 128;
        pl.kernel = kKSplit;
        int off = 0;
        auto take = [&](int64_t bytes) { const int o_ = off; off += (int)align_up(bytes, 16); return o_; };
        pl.off_q = take(4LL * ix->dim);
        pl.off_wl = take(8LL * t);
        pl.off_sk = take(8LL * srpad);
        pl.off_nk = take(8LL * srpad);
        pl.off_fid = take(2LL * align_up(t, 8) + 2LL * srpad);  // merge ranks (int16)
        pl.off_code = take(16LL * srpad);  // the row keys, double-buffered
        // staged code rows (16*MV bytes each); the replay records reuse it
        pl.off_dup = take(std::max<int64_t>(16LL * mv * srpad, 10LL * srpad));
        pl.off_alive = take(srpad);        // replay output
        pl.off_hrow = take(4LL * srpad);   // the head's row ids, staged by the list warps
        pl.off_acc = take(256);            // SplitMisc
        pl.off_vis = take(t);
        pl.off_tab = take(tab_bytes);
        pl.per_warp = off;
        pl.shared_bytes = 0;
        pl.warps = pl.nt / 32;
        pl.smem = off;
        if (pl.smem > ix->max_smem) return fail(BANG_E_PARAM, "t=%d: %d B of shared memory per query", t, pl.smem);
        pl.fn = pick_split_kernel(spl, pl.sub, pl.mv);
        if (!pl.fn) return fail(BANG_E_STATE, "no split kernel for pl=%d sub=%d mv=%d", spl, pl.sub, pl.mv);
        CU(cudaFuncSetAttribute(pl.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem));
        int per_sm = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pl.fn, pl.nt, pl.smem));
        if (per_sm < 1) return fail(BANG_E_CUDA, "search CTA cannot be resident");
        pl.ctas = (int)std::min<int64_t>((int64_t)ix->sm_count * per_sm, std::max<int64_t>(1, nq));
        pl.slots = pl.ctas;
        return BANG_OK;
    }
    // ---- one CTA per query (search_cta_kernel)
    if (!forced_generic && mv > 0) {
        pl.variant = kAdcSmemTable;
        pl.sub = vsub;
        pl.mv = mv;
        pl.nt = 2 * rpad;
        if (t > 4 * 2 * rpad)
            return fail(BANG_E_PARAM, "t=%d exceeds the CTA kernel's worklist limit %d", t, 8 * rpad);
        pl.kernel = kKCta;
        int off = 0;
        auto take = [&](int64_t bytes) { const int o_ = off; off += (int)align_up(bytes, 16); return o_; };
        pl.off_q = take(4LL * ix->dim);
        pl.off_wl = take(8LL * t);
        pl.off_sk = take(8LL * rpad);
        pl.off_nk = take(8LL * rpad);
        pl.off_fid = take(4LL * rpad);
        pl.off_alive = take(rpad);
        pl.off_acc = take(256);  // CtaMisc
        pl.off_vis = take(t);
        pl.off_sum = take(4LL * pl.sum_words);
        pl.off_tab = take(tab_bytes);
        if (ix->row_hdr) pl.off_row = take(4LL * (rpad + 4));
        pl.per_warp = off;  // bytes per CTA
        pl.shared_bytes = 0;
        pl.warps = pl.nt / 32;
        pl.smem = pl.per_warp;
        if (pl.smem > ix->max_smem) return fail(BANG_E_PARAM, "t=%d: %d B of shared memory per query", t, pl.smem);
        pl.fn = pick_cta_kernel(pl.nt, pl.sub, pl.mv, ix->row_hdr);
        if (!pl.fn) return fail(BANG_E_STATE, "no CTA kernel for nt=%d sub=%d mv=%d", pl.nt, pl.sub, pl.mv);
        CU(cudaFuncSetAttribute(pl.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem));
        int per_sm = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pl.fn, pl.nt, pl.smem));
        if (per_sm < 1) return fail(BANG_E_CUDA, "search CTA cannot be resident");
        pl.ctas = (int)std::min<int64_t>((int64_t)ix->sm_count * per_sm, std::max<int64_t>(1, nq));
        pl.slots = pl.ctas;
        return BANG_OK;
    }
    // ---- one warp per query (search_kernel).  Per-warp shared memory: query,
    // worklist keys, sorted/unsorted new keys, fresh ids, partial ADC sums,
    // alive list, visited flags, Bloom summary (one bit per u32 filter word)
    pl.kernel = kKGeneric;
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
    pl.off_tab = pl.per_warp;
    if (pl.variant == kAdcSmemTable) pl.per_warp += (int)tab_bytes;
    pl.shared_bytes = pl.variant == kAdcSmemCodebook ? (int)cb_shared : 0;
    pl.sub = (pl.variant == kAdcSmemCodebook || pl.variant == kAdcSmemTable) ? vsub : 0;
    pl.mv = (pl.sub || pl.variant == kAdcGlobalTable) ? mv : 0;
    int64_t w = (ix->max_smem - pl.shared_bytes) / pl.per_warp;
    if (w < 1) return fail(BANG_E_PARAM, "t=%d needs %d B of shared memory per query", t, pl.per_warp);
    pl.warps = (int)std::min<int64_t>(kMaxSearchThreads / 32, w);
    pl.smem = pl.shared_bytes + pl.warps * pl.per_warp;
    pl.fn = pick_kernel(pl.npl, pl.sub, pl.mv);
    if (!pl.fn) return fail(BANG_E_STATE, "no kernel instance for npl=%d sub=%d mv=%d", pl.npl, pl.sub, pl.mv);
    CU(cudaFuncSetAttribute(pl.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem));
    int per_sm = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pl.fn, pl.warps * 32, pl.smem));
    while (pl.warps > 1 && per_sm < 1) {  // registers: shrink the CTA until it fits
        pl.warps = pl.warps / 2;
        pl.smem = pl.shared_bytes + pl.warps * pl.per_warp;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pl.fn, pl.warps * 32, pl.smem));
    }
    if (per_sm < 1) return fail(BANG_E_CUDA, "search kernel cannot be resident");
    pl.ctas = (int)std::min<int64_t>((int64_t)ix->sm_count * per_sm, std::max<int64_t>(1, ceil_div(nq, pl.warps)));
    pl.slots = pl.ctas * pl.warps;
    return BANG_OK;
}

// L2 persistence of the Bloom filters: the device-wide carve-out is shared by
// every index on the device; the first index to set it records the previous
// limit, the last one destroyed resets the persisting lines and restores it.
struct PersistState {
    int users = 0;
    size_t prev_limit = 0;
    size_t limit = 0;
};
std::mutex g_persist_mu;
std::map<int, PersistState> g_persist;

bang_status persist_acquire(bang_index *ix, size_t want) {
    std::lock_guard<std::mutex> lk(g_persist_mu);
    PersistState &ps = g_persist[ix->device];
    if (!ix->persist_user) {
        if (ps.users == 0) {
            CU(cudaDeviceGetLimit(&ps.prev_limit, cudaLimitPersistingL2CacheSize));
            ps.limit = ps.prev_limit;
        }
        ++ps.users;
        ix->persist_user = true;
    }
    if (want > ps.limit) {
        CU(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
        ps.limit = want;
    }
    ix->persist_set = ps.limit;
    return BANG_OK;
}

void persist_release(bang_index *ix) {
    if (!ix->persist_user) return;
    std::lock_guard<std::mutex> lk(g_persist_mu);
    PersistState &ps = g_persist[ix->device];
    ix->persist_user = false;
    if (--ps.users == 0) {
        cudaCtxResetPersistingL2Cache();
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, ps.prev_limit);
        cudaGetLastError();
        g_persist.erase(ix->device);
    }
}

// Enqueue one search pass.  Outputs are indexed by query id; log rows by
// pass index when qmap != nullptr.
bang_status launch_pass(bang_index *ix, const Plan &pl, const float *d_queries, int64_t nq_pass,
                        const int32_t *d_qmap, int k, int t, int64_t z, int flags, int32_t *d_ids,
                        float *d_dists, int32_t *d_iters, uint8_t *d_short, int32_t *d_log,
                        int64_t log_cap, const float *d_table, cudaStream_t st) {
    if (ix->bloom.reserve((size_t)pl.slots * pl.bloom_stride)) return BANG_E_OOM;
    if (ix->rr.reserve((size_t)pl.slots * log_cap)) return BANG_E_OOM;
    const bang_options &o = ix->opts;
    const bool cta = pl.kernel == kKCta || pl.kernel == kKSplit;
    SearchParams p{};
    p.codes = ix->codes;
    p.code_stride = ix->code_stride;
    p.centroids = ix->centroids;
    p.sub_off = ix->d_sub_off;
    p.sub_size = ix->d_sub_size;
    p.table = d_table;
    p.adj = ix->adj;
    p.adj_stride = ix->adj_stride;
    p.row_hdr = ix->row_hdr ? 1 : 0;
    p.host_graph = ix->host_graph ? 1 : 0;
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
    p.profile = (flags & BANG_PROFILE_PHASES) ? (o.profile == 2 || o.profile == 3 ? o.profile : 1) : 0;
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
    p.off_dup = pl.off_dup;
    p.bloom_clear = o.bloom_clear != 0;
    p.off_code = pl.off_code;
    p.off_hrow = pl.off_hrow;
    p.head_row = o.head_row != 0;
    p.row_prefetch = o.row_prefetch != 0;
    p.deg_share = pl.kernel == kKSplit && o.bloom_direct && ix->row_share_z == z ? ix->row_share.p : nullptr;
    // reset the per-pass counters (next-query, stats, overflow) but keep t0
    CU(cudaMemsetAsync(ix->counters.p, 0, sizeof(unsigned long long) * kCtrT0, st));
    CU(cudaMemsetAsync(ix->counters.p + kCtrPhase0, 0, sizeof(unsigned long long) * 8, st));
    void *args[] = {&p};
    const dim3 grid(pl.ctas), block(cta ? pl.nt : pl.warps * 32);
    // The per-slot Bloom filters (C2: 888 x 50 KB, C3: 592 x 50 KB) are the
    // search's only re-read random working set; the code/adjacency/vector
    // gathers stream past them.  Mark the filters L2-persisting for this
    // launch (bang_options.l2_persist) so Bloom words stay L2 hits.
    const size_t bloom_bytes = (size_t)pl.slots * pl.bloom_stride * 4;
    if (ix->persist_max > 0 && o.l2_persist) {
        bang_status s = persist_acquire(ix, std::min<size_t>(bloom_bytes, (size_t)ix->persist_max));
        if (s) return s;
        const size_t win = std::min<size_t>(bloom_bytes, (size_t)ix->window_max);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = block;
        cfg.dynamicSmemBytes = (size_t)pl.smem;
        cfg.stream = st;
        cudaLaunchAttribute attr{};
        attr.id = cudaLaunchAttributeAccessPolicyWindow;
        attr.val.accessPolicyWindow.base_ptr = ix->bloom.p;
        attr.val.accessPolicyWindow.num_bytes = win;
        // a window larger than the carve-out would thrash the persisting set
        attr.val.accessPolicyWindow.hitRatio = std::min(1.0f, (float)((double)ix->persist_set / (double)win));
        attr.val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr.val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        CU(cudaLaunchKernelExC(&cfg, pl.fn, args));
        return BANG_OK;
    }
    CU(cudaLaunchKernel(pl.fn, grid, block, args, (size_t)pl.smem, st));
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

// The per-(index, z) bitset of rows with in-row Bloom slot sharing
// (row_share_kernel), built on the first split search at this z.
bang_status ensure_row_share(bang_index *ix, int64_t z, cudaStream_t st) {
    if (ix->row_share_z == z) return BANG_OK;
    bang_status s = ix->row_share.reserve((size_t)ix->n);
    if (s) return s;
    BloomGeom g;
    g.z = (uint64_t)z;
    g.magic = ~0ull / (uint64_t)z;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(ix->n, kShareWarps), (int64_t)ix->sm_count * 16));
    row_share_kernel<<<(unsigned)blocks, 32 * kShareWarps, sizeof(uint32_t) * kShareWarps * 2 * ix->R, st>>>(
        ix->adj, ix->adj_stride, ix->deg, ix->n, ix->R, g, ix->row_share.p);
    CU(cudaGetLastError());
    ix->row_share_z = z;
    return BANG_OK;
}

bang_status enqueue_search(bang_index *ix, const float *d_queries, int64_t nq, int k, int t,
                           int64_t z, int flags, int32_t *d_ids, float *d_dists, int32_t *d_iters,
                           uint8_t *d_short, cudaStream_t st) {
    Plan pl;
    bang_status s = make_plan(ix, nq, t, z, flags, pl);
    if (s) return s;
    const int64_t cap = default_log_cap(ix, t);
    if ((s = ensure_outputs(ix, nq, k, cap))) return s;
    if (pl.kernel == kKSplit && ix->opts.bloom_direct && (s = ensure_row_share(ix, z, st))) return s;
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
    ix->k_last = k;
    ix->stats.slots = pl.slots;
    ix->stats.warps_per_cta = pl.warps;
    ix->stats.ctas = pl.ctas;
    ix->stats.adc_variant = pl.variant;
    ix->stats.kernel = pl.kernel;
    ix->last_nq = nq;
    ix->last_log_cap = cap;
    ix->last_has_table = d_table != nullptr;
    ix->last_rerank = (flags & BANG_RERANK) != 0;
    ix->last_stream = st;
    ix->pending = true;
    return BANG_OK;
}

// Reads counters after the stream drained; fills stats.
bang_status collect_stats(bang_index *ix, const unsigned long long *ctr);

bang_status collect(bang_index *ix, unsigned long long *ctr) {
    CU(cudaStreamSynchronize(ix->last_stream));
    CU(cudaMemcpy(ctr, ix->counters.p, sizeof(unsigned long long) * kCtrCount, cudaMemcpyDeviceToHost));
    return collect_stats(ix, ctr);
}

// search statistics from counters already on the host (the stream is idle)
bang_status collect_stats(bang_index *ix, const unsigned long long *ctr) {
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
    // SURVEY.md 8(d) "whole search" bytes: per query-iteration
    // the adjacency row + degree (4R + 4), per probe its id and two u64 Bloom
    // words (20), per fresh neighbour its code row, id and key (m + 12); per
    // re-rank candidate its vector + id + key; per query the query in and
    // the k results out
    S.algorithmic_bytes = S.iterations * (4LL * ix->R + 4) + S.probes * 20 + S.fresh * (ix->m + 12) +
                          S.rerank_cands * (ix->dim * elem + 12) + S.queries * (ix->dim * 4 + 8LL * ix->k_last);
    S.adc_bytes = S.fresh * (ix->m + 12);
    for (int i = 0; i < 8; ++i) S.phase_cycles[i] = (int64_t)ctr[kCtrPhase0 + i];
    ix->pending = false;
    return BANG_OK;
}

}  // namespace

// ---- PCIe read roofline for the host-resident graph path (diagnostic):
// streaming (mode 0: each thread reads consecutive 16-byte pieces) or random
// rows of row_bytes (mode 1: one warp per row, the search's access pattern)
// from pinned, mapped host memory
__global__ void host_read_kernel(const uint4 *__restrict__ src, int64_t n16, int mode, int row16, int64_t nrows,
                                 int64_t reads, unsigned long long *sink) {
    uint32_t acc = 0;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    if (mode == 0) {
        for (int64_t i = tid; i < n16; i += nt) {
            const uint4 v = src[i];
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    } else {
        const int64_t warp = tid >> 5, nw = nt >> 5;
        const int lane = threadIdx.x & 31;
        for (int64_t r = warp; r < reads; r += nw) {
            const uint64_t h = (uint64_t)r * 0x9E3779B97F4A7C15ull;
            const int64_t row = (int64_t)((h >> 17) % (uint64_t)nrows);
            if (lane < row16) {
                const uint4 v = src[row * row16 + lane];
                acc ^= v.x ^ v.y ^ v.z ^ v.w;
            }
        }
    }
    if (acc == 0x9E3779B9u) atomicAdd(sink, 1ull);  // keeps the loads
}

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
    bang_options_default(&ix->opts);
    // m = 48 code rows are padded to 64 bytes: a gathered row is then one
    // aligned 64-byte DRAM burst instead of straddling two
    ix->code_stride = m == 48 ? 64 : m;
    if (m > 0) {
        CUX(cudaMalloc(&ix->codes, (size_t)n * ix->code_stride));
        if (ix->code_stride == m) {
            CUX(cudaMemcpy(ix->codes, codes, (size_t)n * m, cudaMemcpyHostToDevice));
        } else {
            CUX(cudaMemset(ix->codes, 0, (size_t)n * ix->code_stride));
            CUX(cudaMemcpy2D(ix->codes, ix->code_stride, codes, m, m, n, cudaMemcpyHostToDevice));
        }
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
            // header + row per node, written by all host threads (27 GB at 100M x 64)
            const int T = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
            auto fill = [&](int tix) {
                for (int64_t i = n * tix / T; i < n * (tix + 1) / T; ++i) {
                    int32_t *row = ix->adj_alloc + i * ix->adj_stride;
                    row[0] = degrees[i];
                    row[1] = row[2] = row[3] = 0;
                    memcpy(row + 4, adjacency + i * R, (size_t)R * 4);
                }
            };
            std::vector<std::thread> pool;
            for (int tix = 1; tix < T; ++tix) pool.emplace_back(fill, tix);
            fill(0);
            for (auto &th : pool) th.join();
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
    persist_release(ix);
    cudaFree(ix->codes);
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
    if (ix->h_ctr) cudaFreeHost(ix->h_ctr);
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
    ix->row_share.release();
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
    // the queries' finiteness (validation.py:17-19) is checked on the device,
    // next to the search, instead of by a host pass over them
    CU(cudaMemsetAsync(ix->counters.p + kCtrNonFinite, 0, sizeof(unsigned long long), st));
    {
        const int64_t cnt = nq * ix->dim;
        const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cnt, 256), (int64_t)ix->sm_count * 8));
        check_finite_kernel<<<blocks, 256, 0, st>>>(ix->q.p, cnt, ix->counters.p);
        CU(cudaGetLastError());
    }
    if ((s = enqueue_search(ix, ix->q.p, nq, k, t, bloom_entries, flags, ix->ids.p, ix->dists.p, ix->iters.p,
                            ix->shortf.p, st)))
        return s;
    // One-batch readback when the caller's visit-log buffer is page-locked
    // and holds the worst case (nq x log capacity): offsets scanned and logs
    // compacted on the device straight into it, every output and the
    // counters copied back in one batch, one synchronisation.  An overflowed
    // visit log falls back to the exact re-run below.
    {
        const int64_t cap = ix->last_log_cap;
        cudaPointerAttributes va{};
        const bool direct = visit_ids && visit_offsets && visit_cap >= nq * cap &&
                            cudaPointerGetAttributes(&va, visit_ids) == cudaSuccess &&
                            (va.type == cudaMemoryTypeHost || va.type == cudaMemoryTypeDevice ||
                             va.type == cudaMemoryTypeManaged) && va.devicePointer;
        cudaGetLastError();
        if (direct) {
            if (!ix->h_ctr) CU(cudaHostAlloc(reinterpret_cast<void **>(&ix->h_ctr), sizeof(unsigned long long) * kCtrCount,
                                            cudaHostAllocDefault));
            if ((s = ix->offs.reserve((size_t)nq + 1))) return s;
            scan_offsets_kernel<<<1, 1024, 0, st>>>(ix->iters.p, nq, ix->offs.p);
            compact_logs_kernel<<<(unsigned)ceil_div(nq, 8), 256, 0, st>>>(
                ix->log.p, cap, nq, nullptr, ix->offs.p, nullptr, static_cast<int32_t *>(va.devicePointer));
            CU(cudaGetLastError());
            std::vector<uint64_t> wns(wall ? nq : 0);
            CU(cudaMemcpyAsync(ix->h_ctr, ix->counters.p, sizeof(unsigned long long) * kCtrCount,
                               cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(ids, ix->ids.p, sizeof(int32_t) * nq * k, cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(dists, ix->dists.p, sizeof(float) * nq * k, cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(iterations, ix->iters.p, sizeof(int32_t) * nq, cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(visit_offsets, ix->offs.p, sizeof(int64_t) * (nq + 1), cudaMemcpyDeviceToHost, st));
            if (short_) CU(cudaMemcpyAsync(short_, ix->shortf.p, nq, cudaMemcpyDeviceToHost, st));
            if (wall) CU(cudaMemcpyAsync(wns.data(), ix->wall.p, sizeof(uint64_t) * nq, cudaMemcpyDeviceToHost, st));
            CU(cudaStreamSynchronize(st));
            if ((s = collect_stats(ix, ix->h_ctr))) return s;
            if (ix->h_ctr[kCtrNonFinite]) return fail(BANG_E_PARAM, "queries contains non-finite values");
            if (ix->h_ctr[kCtrDebugFail])
                return fail(BANG_E_STATE, "debug check failed: eager candidate disagrees with the post-merge worklist head");
            if (!ix->h_ctr[kCtrOverflow]) {
                if (converged) memset(converged, 1, nq);  // the loop runs every query to convergence
                if (wall)
                    for (int64_t i = 0; i < nq; ++i) wall[i] = (double)wns[i] * 1e-9;
                ix->last_iters.assign(iterations, iterations + nq);
                ix->last_offsets.assign(visit_offsets, visit_offsets + nq + 1);
                ix->pending = false;
                return BANG_OK;
            }
            // an overflowed log: redo the readback the general way
        }
    }
    unsigned long long ctr[kCtrCount];
    if ((s = collect(ix, ctr))) return s;
    if (ctr[kCtrNonFinite]) return fail(BANG_E_PARAM, "queries contains non-finite values");
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

void bang_options_default(bang_options *o) {
    if (!o) return;
    *o = bang_options{};
    o->kernel = BANG_KERNEL_AUTO;
    o->row_prefetch = 1;
    o->bloom_clear = 1;
    o->l2_persist = 1;
    o->profile = 0;
    o->bloom_direct = 1;
    o->head_row = 1;
}

bang_status bang_index_set_options(bang_index *ix, const bang_options *o) {
    if (!ix || !o) return fail(BANG_E_STATE, "null argument");
    if (o->kernel < BANG_KERNEL_AUTO || o->kernel > BANG_KERNEL_SPLIT || o->kernel == 3)
        return fail(BANG_E_PARAM, "unknown kernel %d", o->kernel);
    ix->opts = *o;
    return BANG_OK;
}

bang_status bang_index_get_options(const bang_index *ix, bang_options *o) {
    if (!ix || !o) return fail(BANG_E_STATE, "null argument");
    *o = ix->opts;
    return BANG_OK;
}

int32_t bang_index_code_stride(const bang_index *ix) { return ix ? ix->code_stride : 0; }

bang_status bang_index_prepare(bang_index *ix, int64_t z) {
    if (!ix) return fail(BANG_E_STATE, "GraphSearcher is not fitted (null index)");
    if (z < 1 || z >= (1LL << 31)) return fail(BANG_E_PARAM, "bloom_entries must be in [1, 2^31), got %lld", (long long)z);
    if (!ix->opts.bloom_direct || ix->m <= 0) return BANG_OK;
    CU(cudaSetDevice(ix->device));
    bang_status s = ensure_row_share(ix, z, ix->stream);
    if (s) return s;
    CU(cudaStreamSynchronize(ix->stream));
    return BANG_OK;
}

// ------------------------------------------------------------ per-kernel entries

bang_status bang_pq_table(bang_index *ix, const float *queries, int64_t nq, float *out) {
    if (!ix) return fail(BANG_E_STATE, "GraphSearcher is not fitted (null index)");
    if (ix->m < 1) return fail(BANG_E_PARAM, "index has no PQ codebook");
    if (nq < 0) return fail(BANG_E_PARAM, "nq must be >= 0");
    if (nq == 0) return BANG_OK;
    if (!queries || !out) return fail(BANG_E_PARAM, "NULL queries/out");
    CU(cudaSetDevice(ix->device));
    cudaStream_t st = ix->stream;
    bang_status s;
    if ((s = ix->q.reserve((size_t)nq * ix->dim))) return s;
    if ((s = ix->table.reserve((size_t)nq * ix->m * 256))) return s;
    CU(cudaMemcpyAsync(ix->q.p, queries, sizeof(float) * nq * ix->dim, cudaMemcpyHostToDevice, st));
    pq_table_kernel<<<(unsigned)nq, 256, ix->dim * sizeof(float), st>>>(ix->centroids, ix->d_sub_off, ix->d_sub_size,
                                                                       ix->m, ix->dim, ix->q.p, ix->table.p);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(out, ix->table.p, sizeof(float) * nq * ix->m * 256, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return BANG_OK;
}

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
    const bool vec = (sub == 4 && mv == 2) || (sub == 2 && mv == 3);
    // table + query (+ per-warp double-buffered code-row stages, vector path)
    constexpr int NT = BANG_ADC_PAIRS_NT;  // threads per query CTA
    const size_t smem = sizeof(float) * ((size_t)ix->m * 256 + align_up(ix->dim, 4)) +
                        (vec ? (size_t)(NT / 32) * 2 * 32 * ix->m : 0);
    if (smem > (size_t)ix->max_smem) return fail(BANG_E_PARAM, "table of m=%d does not fit in shared memory", ix->m);
    auto launch = [&](const void *fn) -> bang_status {
        CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, smem));
        const int64_t grid = std::min<int64_t>(nq, (int64_t)ix->sm_count * std::max(1, per_sm));
        int m = ix->m, dim = ix->dim, cs = ix->code_stride;
        void *args[] = {&ix->centroids, &ix->d_sub_off, &ix->d_sub_size, &m, &dim, &d_queries, &nq,
                        &d_off, &d_ids, &ix->codes, &cs, &d_keys};
        CU(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(NT), args, smem, st));
        return BANG_OK;
    };
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

bang_status bang_host_read_bandwidth(int32_t device, int64_t bytes, int32_t mode, int32_t row_bytes, double *gbs) {
    if (!gbs || bytes < (1 << 20) || (mode != 0 && mode != 1) || (mode == 1 && (row_bytes < 16 || row_bytes > 512 ||
                                                                                row_bytes % 16)))
        return fail(BANG_E_PARAM, "bytes >= 1 MiB, mode 0/1, row_bytes a multiple of 16 in [16, 512]");
    CU(cudaSetDevice(device));
    void *h = nullptr;
    unsigned long long *sink = nullptr;
    CU(cudaHostAlloc(&h, (size_t)bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    memset(h, 1, (size_t)bytes);
    void *d = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(&d, h, 0);
    if (e == cudaSuccess) e = cudaMalloc(&sink, sizeof(unsigned long long));
    cudaEvent_t a = nullptr, b = nullptr;
    if (e == cudaSuccess) e = cudaEventCreate(&a);
    if (e == cudaSuccess) e = cudaEventCreate(&b);
    float ms = 0.0f;
    int64_t moved = 0;
    if (e == cudaSuccess) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        const int64_t n16 = bytes / 16, row16 = row_bytes / 16, nrows = bytes / (row_bytes ? row_bytes : 16);
        const int64_t reads = mode == 1 ? nrows : 0;
        moved = mode == 0 ? n16 * 16 : reads * row_bytes;
        for (int it = 0; it < 2 && e == cudaSuccess; ++it) {  // warm-up, then timed
            cudaEventRecord(a);
            host_read_kernel<<<sms * 8, 256>>>(static_cast<const uint4 *>(d), n16, mode, (int)row16, nrows, reads,
                                               sink);
            cudaEventRecord(b);
            e = cudaEventSynchronize(b);
        }
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, a, b);
    }
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    if (sink) cudaFree(sink);
    cudaFreeHost(h);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(BANG_E_CUDA, "host read bandwidth: %s", cudaGetErrorString(e));
    }
    *gbs = moved / (ms * 1e6);
    return BANG_OK;
}

}  // extern "C"
