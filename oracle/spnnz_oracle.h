/*
 * spnnz CPU oracle -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference predictor hot path
 * (/root/reference/proj/include/spnnz/{rng,flop,symbolic,predict}.hpp).
 * It is the checker for the CUDA path: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product library (paper_2207_13848_b200/csrc) never links or calls it.
 *
 * Parity of this restatement is pinned two ways ("Oracle"):
 *   - the reference's own known-answer tests (tests/test_oracle.py), and
 *   - fixtures produced by the reference itself, compiled from its headers
 *     into oracle/_ref/ (tests/golden/make_golden.py).
 *
 * Error convention: functions return 0 on success and ORACLE_EINVAL where the
 * reference throws std::invalid_argument; oracle_last_error() holds the text.
 */
#ifndef SPNNZ_ORACLE_H
#define SPNNZ_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORACLE_OK 0
#define ORACLE_EINVAL 1
#define ORACLE_ENOMEM 2

typedef struct {
    int32_t rows;
    int32_t cols;
    const int64_t* rpt; /* rows + 1 */
    const int32_t* col; /* rpt[rows] */
} oracle_csr;

const char* oracle_last_error(void);

/* SplitMix64, rng.hpp:14-19 / :22-24 / :27-30 / :34-37 */
uint64_t oracle_splitmix_next(uint64_t* state);
double oracle_splitmix_next_double(uint64_t* state);
uint64_t oracle_splitmix_next_below(uint64_t* state, uint64_t bound);
uint64_t oracle_splitmix_fork(uint64_t seed, uint64_t tag);

/* compute_flop, flop.hpp:25-60 */
int oracle_compute_flop(const oracle_csr* a, const oracle_csr* b, int threads,
                        int64_t* flop_per_row, int64_t* total_flop, int64_t* max_flop_row);
/* sampled_flop, flop.hpp:64-74 */
int oracle_sampled_flop(const int64_t* flop_per_row, int64_t num_rows, const int32_t* rows,
                        int64_t n, int64_t* out);

/* make_sample_plan, predict.hpp:34-56.  rows may be NULL (count/p only);
 * otherwise it must hold the clamped sample count. */
int oracle_sample_count(int32_t num_rows, double fraction, int64_t cap, int64_t* n, double* p);
int oracle_make_sample_plan(int32_t num_rows, uint64_t seed, double fraction, int64_t cap,
                            int32_t* rows, int64_t* n, double* p);

/* HashAccumulator::row_nnz, symbolic.hpp:35-60 (table has >= tsize slots) */
int64_t oracle_row_nnz(const oracle_csr* a, const oracle_csr* b, int32_t row, int64_t tsize,
                       int32_t* table, int64_t hash_scale);
/* exact_symbolic, symbolic.hpp:94-118 */
int oracle_exact_symbolic(const oracle_csr* a, const oracle_csr* b, const int64_t* flop_per_row,
                          int64_t max_flop_row, int threads, int64_t* nnz_per_row,
                          int64_t* total_nnz);
/* sampled_symbolic, symbolic.hpp:122-154 */
int oracle_sampled_symbolic(const oracle_csr* a, const oracle_csr* b, const int64_t* flop_per_row,
                            int64_t max_flop_row, const int32_t* rows, int64_t n, int threads,
                            int64_t* nnz_per_sample, int64_t* total_nnz);

/* Estimators, predict.hpp:81-123 and :163-188 */
double oracle_sampled_cr(int64_t sampled_flop, int64_t sampled_nnz);
int oracle_predict_reference(int64_t sampled_nnz, double p, double* z1);
void oracle_predict_proposed(int64_t sampled_flop, int64_t sampled_nnz, int64_t total_flop,
                             double* z2, double* cr);
typedef struct {
    double eps1, eps_f, eps2, identity_residual;
} oracle_error_report;
int oracle_error_report_compute(double z1, double z2, int64_t f_star, int64_t exact_nnz,
                                int64_t total_flop, double p, oracle_error_report* out);

/* predict_row_structure / _ceil, predict.hpp:126-151 */
int oracle_predict_row_structure(const int64_t* flop_per_row, int64_t m, double cr, double* out);
int oracle_predict_row_structure_ceil(const int64_t* flop_per_row, int64_t m, double cr,
                                      int64_t* out);

/* Whole pipeline, predict.hpp:220-226 plus the ceil view (CLI --structure-out,
 * spnnz_main.cpp:198-199). Outputs mirror PredictionReport. */
typedef struct {
    int64_t total_flop, max_flop_row;
    int64_t sample_num;
    double p;
    int64_t sampled_flop, sampled_nnz;
    double sampled_cr;
    double z1_star, z2_star, predicted_cr;
} oracle_report;
int oracle_run_prediction(const oracle_csr* a, const oracle_csr* b, uint64_t seed,
                          double fraction, int64_t cap, int threads, oracle_report* rep,
                          int64_t* flop_per_row /* M, nullable */,
                          int64_t* row_ceil /* M, nullable */, double* row_real /* nullable */);

#ifdef __cplusplus
}
#endif
#endif
