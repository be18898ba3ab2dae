/*
 * spnnz CPU oracle -- TEST INFRASTRUCTURE ONLY (see spnnz_oracle.h).
 *
 * Plain-C restatement of the reference hot path.  Each function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Build with -ffp-contract=off so the few double expressions round exactly
 * like the reference's (the reference is compiled the same way in oracle/_ref).
 */
#include "spnnz_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static __thread char g_err[256];

static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return ORACLE_EINVAL;
}

const char* oracle_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- rng.hpp */

/* SplitMix64::next_u64, include/spnnz/rng.hpp:14-19 */
uint64_t oracle_splitmix_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* SplitMix64::next_double, rng.hpp:22-24 */
double oracle_splitmix_next_double(uint64_t* state) {
    return (double)(oracle_splitmix_next(state) >> 11) * 0x1.0p-53;
}

/* SplitMix64::next_below (Lemire), rng.hpp:27-30 */
uint64_t oracle_splitmix_next_below(uint64_t* state, uint64_t bound) {
    return (uint64_t)(((unsigned __int128)oracle_splitmix_next(state) * bound) >> 64);
}

/* SplitMix64::fork, rng.hpp:34-37 */
uint64_t oracle_splitmix_fork(uint64_t seed, uint64_t tag) {
    uint64_t s = seed ^ (tag * 0xd1b54a32d192ed03ULL);
    return oracle_splitmix_next(&s);
}

/* ----------------------------------------------------------- parallel.hpp */

/* resolve_threads, include/spnnz/parallel.hpp:12-16 */
static int resolve_threads(int requested) {
    if (requested > 0) return requested;
    long hw = sysconf(_SC_NPROCESSORS_ONLN);
    return hw <= 0 ? 1 : (int)hw;
}

typedef void (*block_fn)(void* ctx, int tid, int64_t begin, int64_t end);

typedef struct {
    block_fn fn;
    void* ctx;
    int tid;
    int64_t begin, end;
} block_job;

static void* block_trampoline(void* p) {
    block_job* j = (block_job*)p;
    j->fn(j->ctx, j->tid, j->begin, j->end);
    return NULL;
}

/* parallel_blocks, parallel.hpp:24-41: block t = [n*t/W, n*(t+1)/W). */
static void parallel_blocks(int64_t n, int workers, block_fn fn, void* ctx) {
    if (n <= 0) return;
    if (workers > n) workers = (int)n;
    if (workers <= 1) {
        fn(ctx, 0, 0, n);
        return;
    }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)workers);
    block_job* jobs = (block_job*)malloc(sizeof(block_job) * (size_t)workers);
    for (int t = 0; t < workers; ++t) {
        jobs[t].fn = fn;
        jobs[t].ctx = ctx;
        jobs[t].tid = t;
        jobs[t].begin = n * t / workers;
        jobs[t].end = n * (t + 1) / workers;
    }
    for (int t = 1; t < workers; ++t) pthread_create(&th[t], NULL, block_trampoline, &jobs[t]);
    block_trampoline(&jobs[0]);
    for (int t = 1; t < workers; ++t) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
}

static int worker_count(int threads, int64_t n) {
    int w = resolve_threads(threads);
    int64_t cap = n > 1 ? n : 1;
    return (int)(w < cap ? w : cap);
}

/* --------------------------------------------------------------- flop.hpp */

typedef struct {
    const oracle_csr *a, *b;
    int64_t* flop;
    int64_t* part_total;
    int64_t* part_max;
} flop_ctx;

/* hot loop, include/spnnz/flop.hpp:41-50 */
static void flop_block(void* p, int tid, int64_t begin, int64_t end) {
    flop_ctx* c = (flop_ctx*)p;
    const int64_t* arpt = c->a->rpt;
    const int32_t* acol = c->a->col;
    const int64_t* brpt = c->b->rpt;
    int64_t tot = 0, mx = 0;
    for (int64_t i = begin; i < end; ++i) {
        int64_t f = 0;
        for (int64_t j = arpt[i]; j < arpt[i + 1]; ++j) {
            const int32_t k = acol[j];
            f += brpt[k + 1] - brpt[k];
        }
        c->flop[i] = f;
        tot += f;
        if (f > mx) mx = f;
    }
    c->part_total[tid] = tot;
    c->part_max[tid] = mx;
}

/* compute_flop, flop.hpp:25-60 */
int oracle_compute_flop(const oracle_csr* a, const oracle_csr* b, int threads,
                        int64_t* flop_per_row, int64_t* total_flop, int64_t* max_flop_row) {
    if (a->cols != b->rows) return fail("compute_flop: A.cols != B.rows"); /* :26-29 */
    const int workers = worker_count(threads, a->rows);
    flop_ctx c = {a, b, flop_per_row, (int64_t*)calloc((size_t)workers, 8),
                  (int64_t*)calloc((size_t)workers, 8)};
    parallel_blocks(a->rows, workers, flop_block, &c);
    int64_t tot = 0, mx = 0; /* serial combine, :55-58 */
    for (int t = 0; t < workers; ++t) {
        tot += c.part_total[t];
        if (c.part_max[t] > mx) mx = c.part_max[t];
    }
    free(c.part_total);
    free(c.part_max);
    *total_flop = tot;
    *max_flop_row = mx;
    return ORACLE_OK;
}

/* sampled_flop, flop.hpp:64-74 (duplicates count once per appearance) */
int oracle_sampled_flop(const int64_t* flop_per_row, int64_t num_rows, const int32_t* rows,
                        int64_t n, int64_t* out) {
    int64_t s = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (rows[i] < 0 || rows[i] >= num_rows) return fail("sampled_flop: row out of range");
        s += flop_per_row[rows[i]];
    }
    *out = s;
    return ORACLE_OK;
}

/* ------------------------------------------------------------ predict.hpp */

/* sample_num = clamp(ceil(fraction * M), 1, cap); p = n / M.  predict.hpp:36-45 */
int oracle_sample_count(int32_t num_rows, double fraction, int64_t cap, int64_t* n, double* p) {
    if (num_rows < 1) return fail("make_sample_plan: M must be >= 1");
    int64_t k = (int64_t)ceil(fraction * (double)num_rows);
    if (k > cap) k = cap;
    if (k < 1) k = 1;
    *n = k;
    *p = (double)k / (double)num_rows;
    return ORACLE_OK;
}

/* make_sample_plan draw loop, predict.hpp:48-54 */
int oracle_make_sample_plan(int32_t num_rows, uint64_t seed, double fraction, int64_t cap,
                            int32_t* rows, int64_t* n, double* p) {
    int rc = oracle_sample_count(num_rows, fraction, cap, n, p);
    if (rc || !rows) return rc;
    uint64_t st = seed;
    for (int64_t r = 0; r < *n; ++r) {
        const double u = oracle_splitmix_next_double(&st);
        int32_t rid = (int32_t)((double)num_rows * u);
        if (rid >= num_rows) rid = num_rows - 1;
        rows[r] = rid;
    }
    return ORACLE_OK;
}

/* ----------------------------------------------------------- symbolic.hpp */

/* HashAccumulator::row_nnz, symbolic.hpp:35-60 */
int64_t oracle_row_nnz(const oracle_csr* a, const oracle_csr* b, int32_t row, int64_t tsize,
                       int32_t* table, int64_t hash_scale) {
    if (tsize == 0) return 0;
    for (int64_t s = 0; s < tsize; ++s) table[s] = -1;
    int64_t nnz = 0;
    for (int64_t i = a->rpt[row]; i < a->rpt[row + 1]; ++i) {
        const int32_t brow = a->col[i];
        for (int64_t j = b->rpt[brow]; j < b->rpt[brow + 1]; ++j) {
            const int32_t key = b->col[j];
            int64_t h = ((int64_t)key * hash_scale) % tsize;
            for (;;) {
                if (table[h] == key) break;
                if (table[h] == -1) {
                    table[h] = key;
                    ++nnz;
                    break;
                }
                h = (h + 1) % tsize;
            }
        }
    }
    return nnz;
}

typedef struct {
    const oracle_csr *a, *b;
    const int64_t* flop;
    int64_t max_flop;
    const int32_t* rows; /* NULL: all rows */
    int64_t* out;
    int64_t* part;
} sym_ctx;

/* worker body of exact_symbolic / sampled_symbolic, symbolic.hpp:101-113, :136-149 */
static void sym_block(void* p, int tid, int64_t begin, int64_t end) {
    sym_ctx* c = (sym_ctx*)p;
    int32_t* table = (int32_t*)malloc(sizeof(int32_t) * (size_t)(c->max_flop > 0 ? c->max_flop : 1));
    int64_t tot = 0;
    for (int64_t s = begin; s < end; ++s) {
        const int32_t rid = c->rows ? c->rows[s] : (int32_t)s;
        const int64_t nnz = oracle_row_nnz(c->a, c->b, rid, c->flop[rid], table, 107);
        c->out[s] = nnz;
        tot += nnz;
    }
    c->part[tid] = tot;
    free(table);
}

static int check_sym(const oracle_csr* a, const oracle_csr* b) {
    if (a->cols != b->rows) return fail("symbolic: A.cols != B.rows"); /* symbolic.hpp:81-83 */
    return ORACLE_OK;
}

/* exact_symbolic, symbolic.hpp:94-118 */
int oracle_exact_symbolic(const oracle_csr* a, const oracle_csr* b, const int64_t* flop_per_row,
                          int64_t max_flop_row, int threads, int64_t* nnz_per_row,
                          int64_t* total_nnz) {
    int rc = check_sym(a, b);
    if (rc) return rc;
    const int workers = worker_count(threads, a->rows);
    sym_ctx c = {a, b, flop_per_row, max_flop_row, NULL, nnz_per_row,
                 (int64_t*)calloc((size_t)workers, 8)};
    parallel_blocks(a->rows, workers, sym_block, &c);
    int64_t t = 0;
    for (int w = 0; w < workers; ++w) t += c.part[w];
    free(c.part);
    *total_nnz = t;
    return ORACLE_OK;
}

/* sampled_symbolic, symbolic.hpp:122-154 */
int oracle_sampled_symbolic(const oracle_csr* a, const oracle_csr* b, const int64_t* flop_per_row,
                            int64_t max_flop_row, const int32_t* rows, int64_t n, int threads,
                            int64_t* nnz_per_sample, int64_t* total_nnz) {
    int rc = check_sym(a, b);
    if (rc) return rc;
    for (int64_t s = 0; s < n; ++s) /* :125-131 */
        if (rows[s] < 0 || rows[s] >= a->rows) return fail("sampled_symbolic: row out of range");
    const int workers = worker_count(threads, n);
    sym_ctx c = {a, b, flop_per_row, max_flop_row, rows, nnz_per_sample,
                 (int64_t*)calloc((size_t)workers, 8)};
    parallel_blocks(n, workers, sym_block, &c);
    int64_t t = 0;
    for (int w = 0; w < workers; ++w) t += c.part[w];
    free(c.part);
    *total_nnz = t;
    return ORACLE_OK;
}

/* ------------------------------------------------------------ estimators */

/* collect_sample_stats ratio, predict.hpp:86-89 */
double oracle_sampled_cr(int64_t f, int64_t z) {
    return (f > 0 && z > 0) ? (double)f / (double)z : 1.0;
}

/* predict_reference, predict.hpp:94-99 */
int oracle_predict_reference(int64_t sampled_nnz, double p, double* z1) {
    if (!(p > 0.0)) return fail("predict_reference: p must be positive");
    *z1 = (double)sampled_nnz / p;
    return ORACLE_OK;
}

/* predict_proposed, predict.hpp:109-123 */
void oracle_predict_proposed(int64_t f, int64_t z, int64_t total_flop, double* z2, double* cr) {
    if (f <= 0 || z <= 0) {
        *cr = 1.0;
        *z2 = (double)total_flop;
        return;
    }
    *cr = (double)f / (double)z;
    *z2 = (double)total_flop * (double)z / (double)f;
}

/* error_report, predict.hpp:163-188 */
int oracle_error_report_compute(double z1, double z2, int64_t f_star, int64_t exact_nnz,
                                int64_t total_flop, double p, oracle_error_report* out) {
    if (exact_nnz <= 0 || total_flop <= 0)
        return fail("error_report: relative error undefined for Z = 0 or F = 0");
    if (!(p > 0.0)) return fail("error_report: p must be positive");
    const double z = (double)exact_nnz, f = (double)total_flop;
    const double fs = (double)f_star / p;
    out->eps1 = (z1 - z) / z;
    out->eps_f = (fs - f) / f;
    out->eps2 = (z2 - z) / z;
    out->identity_residual =
        f_star > 0 ? fabs(out->eps2 - (out->eps1 - out->eps_f) / (1.0 + out->eps_f)) : 0.0;
    return ORACLE_OK;
}

/* predict_row_structure, predict.hpp:126-136 */
int oracle_predict_row_structure(const int64_t* flop, int64_t m, double cr, double* out) {
    if (!(cr > 0.0)) return fail("predict_row_structure: predicted_cr must be positive");
    for (int64_t i = 0; i < m; ++i) out[i] = (double)flop[i] / cr;
    return ORACLE_OK;
}

/* predict_row_structure_ceil, predict.hpp:140-151 */
int oracle_predict_row_structure_ceil(const int64_t* flop, int64_t m, double cr, int64_t* out) {
    if (!(cr > 0.0)) return fail("predict_row_structure_ceil: predicted_cr must be positive");
    for (int64_t i = 0; i < m; ++i) {
        const double exact = (double)flop[i] / cr;
        const int64_t c = (int64_t)ceil(exact);
        out[i] = flop[i] < c ? flop[i] : c;
    }
    return ORACLE_OK;
}

/* run_prediction, predict.hpp:220-226 -> run_prediction_with_plan :202-216 */
int oracle_run_prediction(const oracle_csr* a, const oracle_csr* b, uint64_t seed,
                          double fraction, int64_t cap, int threads, oracle_report* rep,
                          int64_t* flop_out, int64_t* row_ceil, double* row_real) {
    memset(rep, 0, sizeof *rep);
    int64_t m = a->rows;
    int64_t* flop = flop_out ? flop_out : (int64_t*)malloc(sizeof(int64_t) * (size_t)(m ? m : 1));
    int rc = oracle_compute_flop(a, b, threads, flop, &rep->total_flop, &rep->max_flop_row);
    int32_t* rows = NULL;
    int64_t* per = NULL;
    if (rc) goto out;
    rc = oracle_sample_count(a->rows, fraction, cap, &rep->sample_num, &rep->p);
    if (rc) goto out;
    rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)rep->sample_num);
    per = (int64_t*)malloc(sizeof(int64_t) * (size_t)rep->sample_num);
    rc = oracle_make_sample_plan(a->rows, seed, fraction, cap, rows, &rep->sample_num, &rep->p);
    if (rc) goto out;
    rc = oracle_sampled_symbolic(a, b, flop, rep->max_flop_row, rows, rep->sample_num, threads,
                                 per, &rep->sampled_nnz);
    if (rc) goto out;
    rc = oracle_sampled_flop(flop, m, rows, rep->sample_num, &rep->sampled_flop);
    if (rc) goto out;
    rep->sampled_cr = oracle_sampled_cr(rep->sampled_flop, rep->sampled_nnz);
    rc = oracle_predict_reference(rep->sampled_nnz, rep->p, &rep->z1_star);
    if (rc) goto out;
    oracle_predict_proposed(rep->sampled_flop, rep->sampled_nnz, rep->total_flop, &rep->z2_star,
                            &rep->predicted_cr);
    if (row_real) rc = oracle_predict_row_structure(flop, m, rep->predicted_cr, row_real);
    if (!rc && row_ceil) rc = oracle_predict_row_structure_ceil(flop, m, rep->predicted_cr, row_ceil);
out:
    free(rows);
    free(per);
    if (!flop_out) free(flop);
    return rc;
}
