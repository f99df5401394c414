/*
 * bang.h -- C-ABI of libbang.so, the B200 (sm_100a) batched graph-search
 * hot path of BANG (arXiv 2401.11324).
 *
 * Plain pointers and sizes only; no torch or CUDA types in the signatures
 * (streams are passed as void* holding a cudaStream_t, NULL = the handle's
 * own stream).  Every entry point returns BANG_OK (0) or a negative
 * bang_status with a message retrievable from bang_last_error() (thread
 * local).  Paths in the citations are relative to the reference package
 * /root/reference/pkg/src/bang/.
 *
 * Two layers:
 *  1. the index handle + batched search that replaces the reference's
 *     GraphSearcher.fit/search seam (engine.py:377-452 -> _search_batch
 *     engine.py:108-270 + build_pq_dist_table pq.py:299-319);
 *  2. one device-pointer entry per hot-path kernel, each replacing one
 *     reference function (used by the function-level parity tests and by
 *     callers that keep their own device buffers).
 */
#ifndef BANG_H
#define BANG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t bang_status;
#define BANG_OK 0
#define BANG_E_PARAM (-1)    /* maps to ParameterError (errors.py:8-9)          */
#define BANG_E_CUDA (-2)     /* CUDA runtime failure -> BangError              */
#define BANG_E_OOM (-3)      /* device allocation failed -> BangError           */
#define BANG_E_CAPACITY (-4) /* caller buffer too small; sizes reported         */
#define BANG_E_STATE (-5)    /* handle misuse / debug-check failure             */
#define BANG_E_FORMAT (-6)   /* malformed index file -> FileFormatError (errors.py:12-13) */
#define BANG_E_TRUNCATED (-7)/* index file ends early -> TruncatedFileError (errors.py:16-17) */

/* vector scalar kinds (validation.py:8 SUPPORTED_SCALARS) */
#define BANG_VEC_F32 0
#define BANG_VEC_U8 1
#define BANG_VEC_I8 2

/* graph placement: engine.py modes "in_memory" / "pipelined" */
#define BANG_GRAPH_HBM 0
#define BANG_GRAPH_HOST_MAPPED 1

/* bang_search flags */
#define BANG_RERANK 1          /* GraphSearcher(rerank=True), engine.py:254-262  */
#define BANG_DEBUG_CHECKS 2    /* GraphSearcher(debug_checks=True), engine.py:169-227 */
#define BANG_EXACT_DISTANCE 4  /* mode="exact_distance", engine.py:120-124,188-193 */
#define BANG_TABLE_GLOBAL 8    /* ADC from a distance table in HBM (kernel 1 first)   */
#define BANG_TABLE_SMEM 16     /* ADC from a per-query table in shared memory         */
#define BANG_CODEBOOK_SMEM 32  /* ADC recomputing entries from a CTA-shared codebook  */
#define BANG_PROFILE_PHASES 64 /* accumulate per-phase cycles (diagnostics, slower)  */
/* (no ADC flag: the per-query smem table when >= 4 queries fit per SM, else
 *  the shared codebook, else the HBM table)                                */

/* Search kernels (bang_options.kernel; bang_search_stats.kernel reports the
 * one that ran as 0 search_kernel, 2 search_cta_kernel, 8 search_split_kernel). */
#define BANG_KERNEL_AUTO 0  /* split for an HBM graph and t <= 256 (m = 32/48), else cta; warp otherwise */
#define BANG_KERNEL_WARP 1  /* search_kernel: one warp per query, every ADC data flow               */
#define BANG_KERNEL_CTA 2   /* search_cta_kernel: one CTA per query, per-query smem table          */
#define BANG_KERNEL_SPLIT 4 /* search_split_kernel: row warps build the next hop's keys while list
                               warps merge the previous hop's (t <= 256)                          */

/* Per-index tuning (bang_index_set_options); every setting gives identical
 * results -- they only move work between warps and memory levels.
 * bang_options_default() fills the measured-best defaults.               */
typedef struct bang_options {
    int32_t kernel;       /* BANG_KERNEL_*                                               */
    int32_t row_prefetch; /* 1: L2 prefetch of the next head's adjacency row (split)      */
    int32_t bloom_clear;  /* 1: search_cta_kernel clears its filter per query; 0: smem
                             summary bitmap of the words this query wrote               */
    int32_t l2_persist;   /* 1: the Bloom filters get an L2-persisting access window      */
    int32_t profile;      /* with BANG_PROFILE_PHASES: 2 = search_split_kernel's row-warp
                             stages, 3 = its list-warp stages                            */
    int32_t bloom_direct; /* 1 (split): rows without in-row Bloom slot sharing (a per-(index,
                             z) bitset, built once) read their pre-state from the fetch-or
                             itself -- no separate pre-state read and no row barrier     */
    int32_t head_row;     /* 1 (split, HBM graph, with bloom_direct): the list warps stage the
                             published head's adjacency row in shared memory for the next hop */
    int32_t reserved[9];
} bang_options;

typedef struct bang_index bang_index;

typedef struct bang_search_stats {
    int64_t queries;          /* queries searched by the last call              */
    int64_t iterations;       /* sum of per-query iterations (expansions)       */
    int64_t probes;           /* Bloom probes (= sum of expanded degrees)       */
    int64_t fresh;            /* admitted neighbours = ADC (query, node) pairs  */
    int64_t rerank_cands;     /* exact distances computed by the re-rank        */
    int64_t retries;          /* queries re-run because a visit log overflowed  */
    int32_t slots;            /* concurrent query slots (warps) of the kernel   */
    int32_t warps_per_cta;
    int32_t ctas;
    int32_t adc_variant;      /* 0 smem codebook, 1 HBM table, 2 exact, 3 smem table */
    float kernel_ms;          /* device time of the fused search kernel(s)      */
    float table_ms;           /* device time of the PQ-table kernel (0 if none)  */
    int64_t algorithmic_bytes;/* HBM bytes the search must move     */
    int64_t adc_bytes;        /* fresh * (m + 12)               */
    int64_t phase_cycles[8];  /* BANG_PROFILE_PHASES: SM cycles per iteration phase,
                                 summed over warps: 0 adjacency wait, 1 expand,
                                 2 Bloom issue, 3 ADC, 4 Bloom resolve, 5 sort +
                                 eager + prefetch, 6 merge + converge, 7 unused */
    int32_t kernel;           /* 0 search_kernel, 2 search_cta_kernel, 6 search_pf_kernel */
    int32_t reserved;
} bang_search_stats;

/* ---------------------------------------------------------------- errors */

/* Message of the last failure on the calling thread ("" if none). */
const char *bang_last_error(void);
/* Library version string. */
const char *bang_version(void);
/* Number of visible CUDA devices (0 when none; never fails). */
int32_t bang_device_count(void);

/* ------------------------------------------------------- index handle
 * Replaces GraphSearcher.fit with prebuilt artifacts (engine.py:377-407,
 * IndexHost engine.py:54-72).  Host pointers are borrowed for the call and
 * copied:
 *   codes      (n, m) u8                    CompressedVectors  pq.py:78-95
 *   centroids  concat over s of (256, sub_sizes[s]) f32  PQCodebook pq.py:37-75
 *   adjacency  (n, R) int32, -1 padded; degrees (n,)   GraphIndex graph.py:23-67
 *   vectors    (n, dim) of vec_dtype: re-rank / exact-distance vectors
 * codes/centroids may be NULL (m = 0) for an exact-distance-only index.
 * graph_placement: BANG_GRAPH_HBM copies adjacency+vectors to HBM;
 * BANG_GRAPH_HOST_MAPPED keeps one pinned, mapped host copy that the
 * kernel reads over PCIe (paper's host-resident graph, "pipelined").     */
bang_status bang_index_create(int32_t device, const uint8_t *codes, int64_t n, int32_t m,
                              const float *centroids, const int32_t *sub_sizes, int32_t dim,
                              const int32_t *adjacency, const int32_t *degrees, int32_t R,
                              int32_t medoid, const void *vectors, int32_t vec_dtype,
                              int32_t graph_placement, bang_index **out);
void bang_index_destroy(bang_index *index);
/* device ordinal, n, m, dim, R of the handle */
bang_status bang_index_info(const bang_index *index, int32_t *device, int64_t *n, int32_t *m,
                            int32_t *dim, int32_t *R);
/* Device pointers owned by the handle (for the per-kernel entries).  With
 * BANG_GRAPH_HOST_MAPPED and R % 4 == 0 the adjacency rows have a stride of
 * R + 4 int32: a 16-byte [deg, 0, 0, 0] header precedes each row.  Code row
 * i starts at codes + i * bang_index_code_stride(index). */
bang_status bang_index_device_ptrs(const bang_index *index, const uint8_t **codes,
                                   const float **centroids, const int32_t **adjacency,
                                   const int32_t **degrees, const void **vectors);
/* Bytes between device code rows: m, except m = 48 rows padded to 64 bytes
 * (one aligned DRAM burst per gathered row). */
int32_t bang_index_code_stride(const bang_index *index);
/* Build the per-(index, bloom_entries) tables of search_split_kernel (each
 * row's degree with its in-row Bloom slot-sharing flag) now instead of on the
 * first search at that Bloom size (bang_options.bloom_direct); synchronous. */
bang_status bang_index_prepare(bang_index *index, int64_t bloom_entries);
/* Tuning of the searches on this handle (kernel choice and the prefetch
 * kernel's data flows); see bang_options.  Results never depend on it. */
void bang_options_default(bang_options *options);
bang_status bang_index_set_options(bang_index *index, const bang_options *options);
bang_status bang_index_get_options(const bang_index *index, bang_options *options);

/* ------------------------------------------------------ batched search
 * GraphSearcher.search for one batch (engine.py:409-452): queries host
 * (nq, dim) f32; outputs host, caller-allocated:
 *   ids (nq,k) int32 -1 padded; dists (nq,k) f32 +inf padded;
 *   iterations (nq) int32; converged (nq) u8; short_ (nq) u8;
 *   wall (nq) f64 seconds from the start of the call (may be NULL);
 *   visit_offsets (nq+1) int64 CSR offsets of the visit logs (may be NULL);
 *   visit_ids[visit_cap] int32 expanded ids in visit order (may be NULL).
 * If visit_ids is non-NULL and the logs need more than visit_cap entries,
 * all other outputs are complete, visit_offsets is filled, and the call
 * returns BANG_E_CAPACITY; fetch the logs with bang_last_visit_logs().
 * k in [1, t]; bloom_entries >= 1 (< 2^31).                              */
bang_status bang_search(bang_index *index, const float *queries, int64_t nq, int32_t k,
                        int32_t t, int64_t bloom_entries, int32_t flags, int32_t *ids,
                        float *dists, int32_t *iterations, uint8_t *converged,
                        uint8_t *short_, double *wall, int64_t *visit_offsets,
                        int32_t *visit_ids, int64_t visit_cap);
/* Copies the visit logs of the last bang_search (CSR order) into visit_ids. */
bang_status bang_last_visit_logs(bang_index *index, int32_t *visit_ids, int64_t visit_cap);
/* Device visit-log capacity per query for the next searches (0 = the
 * default max(1024, 4t)).  Queries that expand more nodes are re-run with a
 * log sized to their exact iteration count; results never depend on it. */
bang_status bang_index_set_log_capacity(bang_index *index, int64_t capacity);
/* Statistics of the last search on this handle. */
bang_status bang_last_search_stats(const bang_index *index, bang_search_stats *out);

/* Device-resident variant (inputs/outputs are device pointers, enqueued on
 * `stream`, no host synchronisation, no visit-log output).  Returns
 * BANG_E_CAPACITY *on the next call or bang_sync_status* if a visit log
 * overflowed the internal capacity (only bang_search retries).            */
bang_status bang_search_device(bang_index *index, const float *d_queries, int64_t nq, int32_t k,
                               int32_t t, int64_t bloom_entries, int32_t flags, int32_t *d_ids,
                               float *d_dists, int32_t *d_iterations, uint8_t *d_short,
                               void *stream);
/* Synchronises the handle's last device search and reports overflow/debug
 * failures (BANG_E_CAPACITY / BANG_E_STATE), filling the stats. */
bang_status bang_sync_status(bang_index *index);

/* ------------------------------------------------------------ index load
 * read_graph (io.py:254-278): the PGIX file ("PGIX", u32 {1, n, R, medoid},
 * then per node u32 len + len u32 ids) is memory-mapped; one serial pass
 * walks the length words, then `threads` host threads (0 = all) copy the ids
 * into the caller's (n, R) int32 adjacency (-1 padded) and degrees (n).
 * Errors as the reference reader's: BANG_E_FORMAT (bad magic/version, degree
 * above R, id out of range, trailing bytes), BANG_E_TRUNCATED (short file),
 * in file order.  Host-only: needs no GPU.                                   */
bang_status bang_read_graph_header(const char *path, int64_t *n, int32_t *R, int32_t *medoid);
bang_status bang_read_graph(const char *path, int32_t *adjacency, int32_t *degrees, int64_t n, int32_t R,
                            int32_t threads);

/* PCIe roofline of the host-resident graph path (diagnostic, no handle):
 * GB/s a kernel reads from `bytes` of pinned, mapped host memory -- mode 0
 * streaming, mode 1 random rows of row_bytes, one warp per row (the search's
 * zero-copy row fetch).  The reference has no counterpart (its graph is in
 * host RAM by construction); bench.py reports the host path against it. */
bang_status bang_host_read_bandwidth(int32_t device, int64_t bytes, int32_t mode, int32_t row_bytes, double *gbs);

/* ---------------------------------------------- per-kernel entries (device pointers) */

/* Kernel 1 with host buffers -- build_pq_dist_table(queries, codebook)
 * (pq.py:299-319) on the handle's codebook: queries (nq, dim) f32 host,
 * out (nq, m, 256) f32 host, caller-allocated. */
bang_status bang_pq_table(bang_index *index, const float *queries, int64_t nq, float *out);

/* Kernel 1 -- build_pq_dist_table (pq.py:284-319): out (nq, m, 256) f32,
 * entry = ((d0*d0 + d1*d1) + ...) in f32 without FMA.  sub_sizes is HOST. */
bang_status bang_pq_table_device(const float *d_centroids, const int32_t *sub_sizes, int32_t m,
                                 int32_t dim, const float *d_queries, int64_t nq, float *d_out,
                                 void *stream);

/* Kernel 2 -- BloomFilterBank.filter_and_set (bloom.py:124-163).
 * d_bits: (count, words64) u64 bank as raw u32 words (2*words64 per row,
 * words64 = ceil(entries/64)).  Probes in CSR order: row r owns
 * [d_row_offsets[r], d_row_offsets[r+1]) of d_ids (low 32 bits of the id,
 * bloom.py:31-33 hashes only those), processed in order.  d_fresh (u8). */
bang_status bang_bloom_filter_device(uint32_t *d_bits, int64_t count, int64_t entries,
                                     const int64_t *d_row_offsets, const uint32_t *d_ids,
                                     uint8_t *d_fresh, void *stream);

/* Kernel 3 -- ADC _pq_point_dists (engine.py:99-105) + pack_keys
 * (kernels.py:25-29): dists[i] = sum_{s<m} table[qrows[i], s, codes[ids[i], s]]
 * sequential f32; keys[i] = f32bits << 32 | ids[i].  Either output may be NULL. */
bang_status bang_adc_device(const float *d_table, int32_t m, const uint8_t *d_codes,
                            const int64_t *d_qrows, const uint32_t *d_ids, int64_t n,
                            float *d_dists, uint64_t *d_keys, void *stream);

/* Kernel 3 over query-grouped pairs: one CTA per query builds
 * its table in shared memory (kernel 1 fused), then keys[i] = pack(ADC(q, ids[i]),
 * ids[i]) for i in [off[q], off[q+1]).  d_queries (nq, dim) f32; d_off (nq+1)
 * int64 non-decreasing; d_keys (off[nq]) u64.  Same arithmetic as
 * bang_adc_device on kernel 1's table (engine.py:99-105, pq.py:284-296). */
bang_status bang_adc_pairs_device(bang_index *index, const float *d_queries, int64_t nq,
                                  const int64_t *d_off, const uint32_t *d_ids, uint64_t *d_keys,
                                  void *stream);

/* Kernel 4a -- merge_sort_rows (kernels.py:94-109): ascending rows, in place. */
bang_status bang_sort_rows_device(uint64_t *d_keys, int64_t rows, int32_t width, void *stream);
/* Kernel 4b -- merge_rows (kernels.py:68-87): out (rows, wa+wb), a first on ties;
 * out_payload takes a_payload (u8, may be NULL) and 0 for b. */
bang_status bang_merge_rows_device(const uint64_t *d_a, const uint8_t *d_a_payload, int64_t rows,
                                   int32_t wa, const uint64_t *d_b, int32_t wb, uint64_t *d_out,
                                   uint8_t *d_out_payload, void *stream);
/* Kernel 4 (engine step) -- eager pick + sort + merge + truncate + converge
 * (engine.py:201-217) for `rows` worklists of width t (keys + u8 visited
 * flags, updated in place) and unsorted new keys (rows, w) SENTINEL-padded:
 * winner[r] = min(min new, min unvisited wl) ; done[r] = all(vis | SENTINEL). */
bang_status bang_worklist_update_device(uint64_t *d_wl_keys, uint8_t *d_wl_vis, int64_t rows,
                                        int32_t t, const uint64_t *d_new_keys, int32_t w,
                                        uint64_t *d_winner, uint8_t *d_done, void *stream);

/* Kernel 5 -- re-rank (engine.py:244-262, 273-292, exact_sq_dists 48-51):
 * per query i the candidates d_cand_ids[d_offsets[i] .. d_offsets[i+1]) in
 * visit order; exact f64-accumulated distances rounded to f32; top-k by
 * (dist, id); ids -1 / dists +inf padded; short = count < k. */
bang_status bang_rerank_device(const void *d_vectors, int32_t vec_dtype, int32_t dim,
                               const float *d_queries, int64_t nq, const int64_t *d_offsets,
                               const int32_t *d_cand_ids, int32_t k, int32_t *d_ids,
                               float *d_dists, uint8_t *d_short, void *stream);
/* exact_sq_dists (engine.py:48-51), row-paired: out[i] = |points[i]-queries[i]|^2 */
bang_status bang_exact_sq_dists_device(const void *d_points, int32_t vec_dtype, int32_t dim,
                                       const float *d_queries, int64_t n, float *d_out,
                                       void *stream);

#ifdef __cplusplus
}
#endif
#endif /* BANG_H */
