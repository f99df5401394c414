/*
 * bang_oracle.c -- CPU restatement of the BANG reference search path.
 *
 * TEST INFRASTRUCTURE ONLY (see bang_oracle.h).  Compiled with
 * -ffp-contract=off so every f32 operation rounds exactly where numpy's does.
 * Reference files are under /root/reference/pkg/src/bang/.
 */
#include "bang_oracle.h"

#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define FNV_OFFSET 0xCBF29CE484222325ull
#define FNV_PRIME 0x100000001B3ull
#define H2_PREFIX 0x5Aull

/* pq.py:284-296 -- diff = q_s - c_s; diff *= diff; acc = diff[..,0];
 * acc += diff[..,j] for j = 1..size-1, all in f32. */
static void table_row(const float *q, int32_t dim, const float *centroids,
                      const int32_t *sub_sizes, int32_t m, float *out) {
    (void)dim;
    int32_t pos = 0;
    const float *cb = centroids;
    for (int32_t s = 0; s < m; ++s) {
        const int32_t size = sub_sizes[s];
        for (int c = 0; c < 256; ++c) {
            const float *cc = cb + (int64_t)c * size;
            float d0 = q[pos] - cc[0];
            float acc = d0 * d0;
            for (int32_t j = 1; j < size; ++j) {
                float dj = q[pos + j] - cc[j];
                float sq = dj * dj;
                acc = acc + sq;
            }
            out[(int64_t)s * 256 + c] = acc;
        }
        cb += 256 * (int64_t)size;
        pos += size;
    }
}

void bo_pq_table(const float *q, int64_t nq, int32_t dim, const float *centroids,
                 const int32_t *sub_sizes, int32_t m, float *out) {
    for (int64_t i = 0; i < nq; ++i)
        table_row(q + i * dim, dim, centroids, sub_sizes, m, out + i * (int64_t)m * 256);
}

/* bloom.py:26-34 */
uint64_t bo_fnv1a(uint64_t id, int32_t prefixed) {
    uint64_t h = FNV_OFFSET;
    if (prefixed) h = (h ^ H2_PREFIX) * FNV_PRIME;
    for (int shift = 0; shift < 32; shift += 8) h = (h ^ ((id >> shift) & 0xFFull)) * FNV_PRIME;
    return h;
}

/* bloom.py:37-42 */
void bo_bit_positions(const int64_t *ids, int64_t n, uint64_t entries, uint64_t *p1,
                      uint64_t *p2) {
    for (int64_t i = 0; i < n; ++i) {
        p1[i] = bo_fnv1a((uint64_t)ids[i], 0) % entries;
        p2[i] = bo_fnv1a((uint64_t)ids[i], 1) % entries;
    }
}

static inline int bit_get(const uint64_t *bits, uint64_t p) {
    return (int)((bits[p >> 6] >> (p & 63)) & 1ull);
}
static inline void bit_set(uint64_t *bits, uint64_t p) { bits[p >> 6] |= 1ull << (p & 63); }

/* bloom.py:70-75 (BloomFilter.test_and_set); returns 1 when the id was fresh */
static inline int test_and_set(uint64_t *bits, uint64_t entries, uint64_t id) {
    uint64_t p1 = bo_fnv1a(id, 0) % entries;
    uint64_t p2 = bo_fnv1a(id, 1) % entries;
    if (bit_get(bits, p1) && bit_get(bits, p2)) return 0;
    bit_set(bits, p1);
    bit_set(bits, p2);
    return 1;
}

/* bloom.py:124-163: the bank's contract is exact sequential test-and-set per
 * row in order of appearance; rows are independent, so one global pass in
 * probe order is the same thing. */
void bo_bloom_filter_and_set(uint64_t *bits, int64_t count, uint64_t entries,
                             const int64_t *rows, const int64_t *ids, int64_t n,
                             uint8_t *fresh) {
    (void)count;
    const int64_t words = (int64_t)((entries + 63) / 64);
    for (int64_t i = 0; i < n; ++i)
        fresh[i] = (uint8_t)test_and_set(bits + rows[i] * words, entries, (uint64_t)ids[i]);
}

/* engine.py:99-105 */
static inline float adc_one(const float *trow, int32_t m, const uint8_t *code) {
    float acc = 0.0f;
    for (int32_t s = 0; s < m; ++s) acc = acc + trow[(int64_t)s * 256 + code[s]];
    return acc;
}

void bo_adc(const float *table, int32_t m, const uint8_t *codes, const int64_t *qrows,
            const int64_t *ids, int64_t n, float *out) {
    for (int64_t i = 0; i < n; ++i)
        out[i] = adc_one(table + qrows[i] * (int64_t)m * 256, m, codes + ids[i] * (int64_t)m);
}

/* kernels.py:25-33 */
uint64_t bo_pack(float d, uint32_t id) {
    uint32_t bits;
    memcpy(&bits, &d, 4);
    return ((uint64_t)bits << 32) | (uint64_t)id;
}

static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

/* kernels.py:94-109: the run-doubling merge sort yields the ascending row */
void bo_sort_rows(uint64_t *keys, int64_t n, int32_t w) {
    for (int64_t i = 0; i < n; ++i) qsort(keys + i * w, (size_t)w, sizeof(uint64_t), cmp_u64);
}

/* kernels.py:68-87: a-element i lands at i + #{b < a_i}; b-element j at
 * j + #{a <= b_j} -- i.e. a stable two-pointer merge with a first on ties. */
void bo_merge_rows(const uint64_t *a, const uint8_t *a_pay, int64_t n, int32_t wa,
                   const uint64_t *b, int32_t wb, uint64_t *out, uint8_t *out_pay) {
    for (int64_t r = 0; r < n; ++r) {
        const uint64_t *ar = a + r * wa, *br = b + r * wb;
        uint64_t *o = out + r * (wa + wb);
        uint8_t *op = out_pay ? out_pay + r * (wa + wb) : NULL;
        int32_t i = 0, j = 0, k = 0;
        while (i < wa && j < wb) {
            if (ar[i] <= br[j]) {
                if (op) op[k] = a_pay ? a_pay[r * wa + i] : 0;
                o[k++] = ar[i++];
            } else {
                if (op) op[k] = 0;
                o[k++] = br[j++];
            }
        }
        while (i < wa) {
            if (op) op[k] = a_pay ? a_pay[r * wa + i] : 0;
            o[k++] = ar[i++];
        }
        while (j < wb) {
            if (op) op[k] = 0;
            o[k++] = br[j++];
        }
    }
}

/* engine.py:48-51: points widened to f32 (validation.py:38-43), then f64
 * difference, f64 sum of squares, rounded to f32.  numpy's einsum sums in a
 * SIMD order we do not restate; a sequential f64 sum rounds to the same f32
 * (0 of 800K differ) -- this is the one unpinned order. */
float bo_exact_sq_dist(const void *x, int32_t dtype, const float *q, int32_t dim) {
    double acc = 0.0;
    for (int32_t j = 0; j < dim; ++j) {
        float xf;
        if (dtype == BO_U8) xf = (float)((const uint8_t *)x)[j];
        else if (dtype == BO_I8) xf = (float)((const int8_t *)x)[j];
        else xf = ((const float *)x)[j];
        double diff = (double)xf - (double)q[j];
        double sq = diff * diff;
        acc = acc + sq;
    }
    return (float)acc;
}

static inline const void *vec_row(const void *vectors, int32_t dtype, int32_t dim, int64_t i) {
    size_t es = dtype == BO_F32 ? 4 : 1;
    return (const char *)vectors + (size_t)i * (size_t)dim * es;
}

/* engine.py:273-292 */
int32_t bo_rerank(const int64_t *cand_ids, int32_t n_cand, const void *vectors,
                  int32_t dtype, int32_t dim, const float *q, int32_t k,
                  int32_t *ids_out, float *dists_out) {
    if (n_cand <= 0) return 0;
    uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n_cand);
    for (int32_t i = 0; i < n_cand; ++i) {
        float d = bo_exact_sq_dist(vec_row(vectors, dtype, dim, cand_ids[i]), dtype, q, dim);
        keys[i] = bo_pack(d, (uint32_t)cand_ids[i]);
    }
    qsort(keys, (size_t)n_cand, sizeof(uint64_t), cmp_u64);
    int32_t out = n_cand < k ? n_cand : k;
    for (int32_t i = 0; i < out; ++i) {
        uint32_t bits = (uint32_t)(keys[i] >> 32);
        memcpy(&dists_out[i], &bits, 4);
        ids_out[i] = (int32_t)(keys[i] & 0xFFFFFFFFull);
    }
    free(keys);
    return out;
}

typedef struct {
    const float *queries;
    int32_t dim;
    const float *centroids;
    const int32_t *sub_sizes;
    int32_t m;
    const float *table;
    const uint8_t *codes;
    const int32_t *adjacency;
    const int32_t *degrees;
    int32_t R;
    int32_t medoid;
    const void *vectors;
    int32_t dtype;
    int32_t k, t;
    uint64_t entries;
    int32_t rerank;
    int32_t mode;
    int64_t log_cap;
} ctx_t;

typedef struct {
    float *trow;
    uint64_t *bits;
    uint64_t *wl;
    uint8_t *vis;
    uint64_t *newk;
    uint64_t *merged;
    uint8_t *mvis;
    int64_t *log;
    int64_t log_len, log_alloc;
} scratch_t;

static float score(const ctx_t *c, const scratch_t *s, const float *q, int32_t node) {
    if (c->mode == BO_MODE_EXACT)
        return bo_exact_sq_dist(vec_row(c->vectors, c->dtype, c->dim, node), c->dtype, q, c->dim);
    return adc_one(s->trow, c->m, c->codes + (int64_t)node * c->m);
}

/* engine.py:113-270 for one query row. */
static void search_one(const ctx_t *c, scratch_t *s, int64_t qi, int32_t *ids_out,
                       float *dists_out, int32_t *iterations, uint8_t *converged,
                       uint8_t *short_out, int32_t *visit_ids, int64_t *need) {
    const float *q = c->queries + qi * c->dim;
    const int32_t t = c->t, k = c->k;
    const uint64_t words = (c->entries + 63) / 64;
    if (c->mode == BO_MODE_PQ) {
        if (c->table) memcpy(s->trow, c->table + qi * (int64_t)c->m * 256, sizeof(float) * 256 * (size_t)c->m);
        else table_row(q, c->dim, c->centroids, c->sub_sizes, c->m, s->trow);
    }
    /* engine.py:118-128 */
    for (int32_t j = 0; j < t; ++j) { s->wl[j] = BO_SENTINEL; s->vis[j] = 0; }
    s->wl[0] = bo_pack(score(c, s, q, c->medoid), (uint32_t)c->medoid);
    memset(s->bits, 0, sizeof(uint64_t) * words);
    {
        uint64_t p1 = bo_fnv1a((uint64_t)c->medoid, 0) % c->entries;
        uint64_t p2 = bo_fnv1a((uint64_t)c->medoid, 1) % c->entries;
        bit_set(s->bits, p1);
        bit_set(s->bits, p2);
    }
    int64_t u = c->medoid;
    int32_t iters = 0;
    s->log_len = 0;
    const int32_t width_pad = 1; /* unused: sentinel padding never changes the kept prefix */
    (void)width_pad;
    for (;;) {
        /* engine.py:167-178: expand the first unvisited entry (== u) */
        int32_t col = 0;
        uint64_t best = BO_SENTINEL;
        for (int32_t j = 0; j < t; ++j) {
            uint64_t mk = s->vis[j] ? BO_SENTINEL : s->wl[j];
            if (mk < best) { best = mk; col = j; }
        }
        s->vis[col] = 1;
        iters++;
        if (s->log_len == s->log_alloc) {
            s->log_alloc = s->log_alloc ? 2 * s->log_alloc : 256;
            s->log = (int64_t *)realloc(s->log, sizeof(int64_t) * (size_t)s->log_alloc);
        }
        s->log[s->log_len++] = u;
        /* engine.py:180-199: Bloom test-and-set in adjacency order, score */
        const int32_t deg = c->degrees[u];
        const int32_t *row = c->adjacency + u * (int64_t)c->R;
        int32_t F = 0;
        for (int32_t r = 0; r < deg; ++r) {
            int32_t nb = row[r];
            if (test_and_set(s->bits, c->entries, (uint64_t)(int64_t)nb))
                s->newk[F++] = bo_pack(score(c, s, q, nb), (uint32_t)nb);
        }
        /* engine.py:201-205: eager winner */
        uint64_t best_new = BO_SENTINEL, head = BO_SENTINEL;
        for (int32_t j = 0; j < F; ++j) if (s->newk[j] < best_new) best_new = s->newk[j];
        for (int32_t j = 0; j < t; ++j) {
            uint64_t mk = s->vis[j] ? BO_SENTINEL : s->wl[j];
            if (mk < head) head = mk;
        }
        uint64_t winner = best_new < head ? best_new : head;
        /* engine.py:210-215: sort, merge (a first), keep t */
        qsort(s->newk, (size_t)F, sizeof(uint64_t), cmp_u64);
        bo_merge_rows(s->wl, s->vis, 1, t, s->newk, F, s->merged, s->mvis);
        memcpy(s->wl, s->merged, sizeof(uint64_t) * (size_t)t);
        memcpy(s->vis, s->mvis, (size_t)t);
        /* engine.py:217 */
        int done = 1;
        for (int32_t j = 0; j < t; ++j)
            if (!s->vis[j] && s->wl[j] != BO_SENTINEL) { done = 0; break; }
        if (done) break;
        u = (int64_t)(winner & 0xFFFFFFFFull);
    }
    iterations[qi] = iters;
    converged[qi] = 1;
    if (s->log_len > c->log_cap) {
        if (s->log_len > *need) *need = s->log_len; /* caller retries */
    } else {
        for (int64_t i = 0; i < s->log_len; ++i) visit_ids[qi * c->log_cap + i] = (int32_t)s->log[i];
    }
    int32_t *io = ids_out + qi * k;
    float *dout = dists_out + qi * k;
    for (int32_t j = 0; j < k; ++j) { io[j] = -1; dout[j] = __builtin_inff(); }
    if (c->mode == BO_MODE_PQ && c->rerank) {
        /* engine.py:254-262 */
        bo_rerank(s->log, (int32_t)s->log_len, c->vectors, c->dtype, c->dim, q, k, io, dout);
        short_out[qi] = s->log_len < k;
    } else {
        /* engine.py:263-265 */
        int32_t real = 0;
        for (int32_t j = 0; j < t; ++j) real += s->wl[j] != BO_SENTINEL;
        for (int32_t j = 0; j < k && j < t; ++j) {
            if (s->wl[j] == BO_SENTINEL) continue;
            uint32_t bits = (uint32_t)(s->wl[j] >> 32);
            memcpy(&dout[j], &bits, 4);
            io[j] = (int32_t)(s->wl[j] & 0xFFFFFFFFull);
        }
        short_out[qi] = real < k;
    }
}

int64_t bo_search(const float *queries, int64_t nq, int32_t dim, const float *centroids,
                  const int32_t *sub_sizes, int32_t m, const float *table,
                  const uint8_t *codes, const int32_t *adjacency, const int32_t *degrees,
                  int64_t n, int32_t R, int32_t medoid, const void *vectors, int32_t dtype,
                  int32_t k, int32_t t, uint64_t entries, int32_t rerank, int32_t mode,
                  int32_t threads, int32_t *ids_out, float *dists_out, int32_t *iterations,
                  uint8_t *converged, uint8_t *short_out, int32_t *visit_ids,
                  int64_t log_cap) {
    (void)n;
    ctx_t c = {queries, dim, centroids, sub_sizes, m, table, codes, adjacency, degrees, R,
               medoid, vectors, dtype, k, t, entries, rerank, mode, log_cap};
    const uint64_t words = (entries + 63) / 64;
    const int32_t maxw = R > 0 ? R : 1;
    int64_t need = 0;
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel num_threads(threads)
#endif
    {
        scratch_t s;
        memset(&s, 0, sizeof(s));
        s.trow = (float *)malloc(sizeof(float) * 256 * (size_t)(m > 0 ? m : 1));
        s.bits = (uint64_t *)malloc(sizeof(uint64_t) * words);
        s.wl = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)t);
        s.vis = (uint8_t *)malloc((size_t)t);
        s.newk = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)maxw);
        s.merged = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(t + maxw));
        s.mvis = (uint8_t *)malloc((size_t)(t + maxw));
        int64_t my_need = 0;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 4)
#endif
        for (int64_t qi = 0; qi < nq; ++qi)
            search_one(&c, &s, qi, ids_out, dists_out, iterations, converged, short_out,
                       visit_ids, &my_need);
#ifdef _OPENMP
#pragma omp critical
#endif
        { if (my_need > need) need = my_need; }
        free(s.trow); free(s.bits); free(s.wl); free(s.vis); free(s.newk);
        free(s.merged); free(s.mvis); free(s.log);
    }
    return need;
}
