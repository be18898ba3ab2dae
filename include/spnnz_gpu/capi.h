/*
 * spnnz_gpu -- C ABI of the B200 SpGEMM output-structure predictor.
 *
 * Drop-in GPU path for the reference's predictor API (namespace spnnz,
 * /root/reference/proj/include/spnnz/{flop,symbolic,predict}.hpp).  Plain
 * pointers and sizes only: no C++ or torch types cross this boundary.
 * Each entry point names the reference function it replaces (file:line,
 * relative to /root/reference/proj).  C++ callers use the header-only mirror
 * include/spnnz_gpu/spnnz_gpu.hpp, which rebuilds the reference's structs and
 * rethrows its exceptions; Python callers use paper_2207_13848_b200.capi.
 *
 * Errors: every function returns SPNNZ_OK (0) or a status code; exceptions
 * cannot cross a C ABI, so the reference's std::invalid_argument becomes
 * SPNNZ_EINVAL with the reference's message in spnnz_gpu_last_error()
 * (thread-local).  There is no CPU fallback: without a usable sm_100 device
 * every device entry point fails with SPNNZ_ECUDA.
 *
 * Multi-GPU: one process (one context) per GPU.  A is row-partitioned into
 * nnz-balanced contiguous shards (spnnz_gpu_partition_rows); B is replicated.
 * Per-row outputs are sharded: rank r owns global rows [row_lo, row_hi) and
 * writes them at local index (row - row_lo).  Totals (F, f*, z*, Z) are
 * combined with one NCCL all-reduce inside the call and are global on every
 * rank.  Per-sample outputs are written for owned samples and 0 elsewhere, so
 * their element-wise sum over ranks is the single-GPU array.
 */
#ifndef SPNNZ_GPU_CAPI_H
#define SPNNZ_GPU_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPNNZ_GPU_ABI_VERSION 1

/* status codes */
#define SPNNZ_OK 0
#define SPNNZ_EINVAL 1 /* reference throws std::invalid_argument */
#define SPNNZ_ECUDA 2  /* CUDA runtime / device error (incl. no GPU) */
#define SPNNZ_ENCCL 3  /* NCCL missing or failed */
#define SPNNZ_ENOMEM 4 /* device or pinned-host allocation failed */
#define SPNNZ_ESTATE 5 /* call order (e.g. no matrices loaded / no profile) */

/* residency of caller buffers */
#define SPNNZ_HOST 0
#define SPNNZ_DEVICE 1

typedef struct spnnz_gpu_ctx spnnz_gpu_ctx;

/* Structure of a CSR matrix: mirrors spnnz::CsrMatrix (include/spnnz/csr.hpp:22-35)
 * without `val`, which no predictor function reads (csr.hpp:12-14).
 * rpt has rows+1 int64 offsets (rpt[0] == 0), col has rpt[rows] int32
 * columns (offset_t / index_t, types.hpp:12-13). */
typedef struct {
    int32_t rows;
    int32_t cols;
    const int64_t* rpt;
    const int32_t* col;
} spnnz_csr_view;

/* Scalars of spnnz::PredictionReport (predict.hpp:192-200) with its
 * SamplePlan (predict.hpp:27-32) and SampleStats (predict.hpp:75-79). */
typedef struct {
    int64_t total_flop;   /* F  (FlopProfile::total_flop) */
    int64_t max_flop_row; /* FlopProfile::max_flop_row */
    int64_t sample_num;   /* SamplePlan::sample_num */
    double p;             /* SamplePlan::p */
    uint64_t seed;        /* SamplePlan::seed */
    int64_t sampled_flop; /* f* */
    int64_t sampled_nnz;  /* z* */
    double sampled_cr;    /* SampleStats::sampled_cr */
    double z1_star;       /* reference design, predict_reference (predict.hpp:94-99) */
    double z2_star;       /* proposed, predict_proposed (predict.hpp:109-123) */
    double predicted_cr;  /* ProposedPrediction::predicted_cr */
} spnnz_report;

/* ------------------------------------------------------------ general */
int spnnz_gpu_abi_version(void);
const char* spnnz_gpu_last_error(void);

/* Fills 128 bytes with an ncclUniqueId (rank 0 calls it and broadcasts). */
int spnnz_gpu_nccl_unique_id(void* id128);

/* One context per GPU. world == 1 needs no NCCL (nccl_id may be NULL; with
 * an id the context joins a one-rank communicator and takes the NCCL path).
 * world > 1 with nccl_id == NULL creates a DETACHED shard: same partition,
 * no communicator, totals stay rank-local and the caller combines them. */
int spnnz_gpu_create(int device, int rank, int world, const void* nccl_id, spnnz_gpu_ctx** out);
int spnnz_gpu_destroy(spnnz_gpu_ctx* ctx);
int spnnz_gpu_synchronize(spnnz_gpu_ctx* ctx);

/* Pinned host buffers for host-residency calls (H2D/D2H at full PCIe rate). */
int spnnz_gpu_host_alloc(size_t bytes, void** out);
int spnnz_gpu_host_free(void* p);

/* Host-only: work-balanced contiguous row shards, bounds[0..world] with
 * bounds[0] = 0 and bounds[world] = rows; shard r = [bounds[r], bounds[r+1]).
 * Work of rows [0, i) = (rpt[i] - rpt[0]) + i (an entry and a row cost about
 * the same in the FLOP and predict passes); bounds[r] = first row i whose
 * work reaches r*(nnz + rows)/world (binary search). */
int spnnz_gpu_partition_rows(const int64_t* rpt, int32_t rows, int world, int32_t* bounds);

/* Upload A (this rank's shard) and B (replicated).  b == NULL or b == a means
 * C = A*A and B shares A's device arrays.  residency says where the view's
 * pointers live.  Throws-equivalent: EINVAL if A.cols != B.rows
 * (flop.hpp:26-29).  Re-loading replaces the previous matrices.
 * Host views are copied asynchronously (for C = A*A in chunks, so the next
 * run_prediction's FLOP pass overlaps the copy): pageable memory is staged
 * before the call returns; pinned memory (spnnz_gpu_host_alloc or
 * cudaHostAlloc) must stay unchanged until the next call on the context
 * returns. */
int spnnz_gpu_load(spnnz_gpu_ctx* ctx, const spnnz_csr_view* a, const spnnz_csr_view* b,
                   int residency);
/* This rank's global A rows [row_lo, row_hi), and the global A.rows. */
int spnnz_gpu_shard(spnnz_gpu_ctx* ctx, int32_t* row_lo, int32_t* row_hi, int32_t* a_rows);

/* ------------------------------------------------- reference functions */

/* spnnz::compute_flop (flop.hpp:25-60).  flop_per_row: this rank's rows
 * (nullable).  total/max are global.  The profile also stays resident in
 * the context for the calls below (FlopProfile argument of the reference). */
int spnnz_gpu_compute_flop(spnnz_gpu_ctx* ctx, int64_t* flop_per_row, int residency,
                           int64_t* total_flop, int64_t* max_flop_row);

/* Install a caller-provided FlopProfile (this rank's rows) as the resident
 * profile, for the reference functions that take `const FlopProfile&`
 * (sampled_flop, sampled_symbolic, exact_symbolic, predict_row_structure*).
 * EINVAL if its length differs from this rank's A rows (symbolic.hpp:84-86). */
int spnnz_gpu_set_profile(spnnz_gpu_ctx* ctx, const int64_t* flop_per_row, int64_t rows,
                          int residency, int64_t total_flop, int64_t max_flop_row);

/* spnnz::sampled_flop (flop.hpp:64-74) over global row ids, duplicates counted.
 * EINVAL on a row outside [0, A.rows).  Needs a resident profile. */
int spnnz_gpu_sampled_flop(spnnz_gpu_ctx* ctx, const int32_t* rows, int64_t n, int residency,
                           int64_t* out);

/* spnnz::make_sample_plan (predict.hpp:34-56), computed on the device.
 * Query form: rows == NULL returns n and p only.  Otherwise rows must hold n
 * entries; indices are identical to the reference's SplitMix64 draws.
 * cap < 0 means "no cap" (INT64_MAX).  EINVAL if num_rows < 1. */
int spnnz_gpu_make_sample_plan(spnnz_gpu_ctx* ctx, int32_t num_rows, uint64_t seed,
                               double fraction, int64_t cap, int32_t* rows, int residency,
                               int64_t* n, double* p);

/* spnnz::sampled_symbolic (symbolic.hpp:122-154): exact output-row NNZ of
 * each sampled row (duplicates recomputed), and the global total z*.
 * nnz_per_sample nullable.  EINVAL on out-of-range rows (:125-131).
 * With a caller-installed profile its flop_per_row is each row's table size,
 * as in the reference: a row whose profile flop is 0 counts 0, and one above
 * the profile's max_flop_row is EINVAL ("HashAccumulator: tsize ... exceeds
 * capacity ...", :37-40); any other row gets its exact count (the
 * reference's probe would not terminate on a table smaller than the row's
 * distinct count; here the count is still exact).  Same for exact_symbolic. */
int spnnz_gpu_sampled_symbolic(spnnz_gpu_ctx* ctx, const int32_t* rows, int64_t n, int residency,
                               int64_t* nnz_per_sample, int64_t* total_nnz);

/* spnnz::exact_symbolic (symbolic.hpp:94-118): exact NNZ of every (owned)
 * output row and the global total Z.  Scoring only (never on the timed path). */
int spnnz_gpu_exact_symbolic(spnnz_gpu_ctx* ctx, int64_t* nnz_per_row, int residency,
                             int64_t* total_nnz);

/* spnnz::predict_row_structure (predict.hpp:126-136) and _ceil (:140-151)
 * over the resident profile; EINVAL unless predicted_cr > 0. */
int spnnz_gpu_predict_row_structure(spnnz_gpu_ctx* ctx, double predicted_cr, double* out,
                                    int residency);
int spnnz_gpu_predict_row_structure_ceil(spnnz_gpu_ctx* ctx, double predicted_cr, int64_t* out,
                                         int residency);

/* spnnz::run_prediction (predict.hpp:220-226) = compute_flop + make_sample_plan
 * + run_prediction_with_plan (:202-216), plus the integer per-row view
 * (predict_row_structure_ceil, as the CLI's --structure-out does,
 * tools/spnnz_main.cpp:198-199).  row_ceil / row_real (this rank's rows) and
 * sample_rows (n entries) are nullable; everything runs on the device with
 * one NCCL all-reduce of {F, f*, z*} when world > 1. */
int spnnz_gpu_run_prediction(spnnz_gpu_ctx* ctx, uint64_t seed, double fraction, int64_t cap,
                             spnnz_report* report, int64_t* row_ceil, double* row_real,
                             int32_t* sample_rows, int residency);

/* spnnz::run_prediction_with_plan (predict.hpp:202-216) on an explicit sample
 * list (e.g. spnnz::exhaustive_plan, :60-70) and the RESIDENT profile -- the
 * reference's `const FlopProfile&` argument: the one compute_flop left, or the
 * caller's installed with set_profile.  No FLOP pass runs: f* and the per-row
 * views come from the profile's flop_per_row, F from its total_flop, and a
 * row's flop is its table size (tsize 0 counts 0; tsize above max_flop_row is
 * EINVAL, symbolic.hpp:35-40).  p is the plan's p.  ESTATE without a profile. */
int spnnz_gpu_run_prediction_with_plan(spnnz_gpu_ctx* ctx, const int32_t* rows, int64_t n, double p,
                                       int rows_residency, spnnz_report* report, int64_t* row_ceil,
                                       double* row_real, int out_residency);

/* The predict step of the reference's harness (bench.hpp:187-195, the task
 * its t_predict times): make_sample_plan + sampled_symbolic +
 * collect_sample_stats + predict_reference + predict_proposed on the
 * RESIDENT profile, in one call (the plan is drawn on the device; no per-row
 * view).  report as run_prediction's; sample_rows (host, n entries) nullable.
 * ESTATE without a profile. */
int spnnz_gpu_predict_sampled(spnnz_gpu_ctx* ctx, uint64_t seed, double fraction, int64_t cap,
                              spnnz_report* report, int32_t* sample_rows);

/* ------------------------------------------- scalar estimators (host) */
/* Same IEEE-double expressions as predict.hpp:86-89, :94-99, :109-123, :163-188. */
double spnnz_sampled_cr(int64_t sampled_flop, int64_t sampled_nnz);
int spnnz_predict_reference(int64_t sampled_nnz, double p, double* z1_star);
int spnnz_predict_proposed(int64_t sampled_flop, int64_t sampled_nnz, int64_t total_flop,
                           double* z2_star, double* predicted_cr);
/* out4 = {eps1, eps_f, eps2, identity_residual} (ErrorReport, predict.hpp:156-161). */
int spnnz_error_report(double z1_star, double z2_star, int64_t f_star, int64_t exact_nnz,
                       int64_t total_flop, double p, double* out4);

/* --------------------------------------------------- instrumentation */
/* Kernel timings of the last run_prediction (ms, CUDA events on the ctx
 * stream, when enabled) and how many of this library's kernels it launched.
 * names: flop, sample, symbolic, allreduce, predict. */
int spnnz_gpu_set_profiling(spnnz_gpu_ctx* ctx, int enabled);
int spnnz_gpu_last_timings(spnnz_gpu_ctx* ctx, double* ms_out5, int64_t* launches);
/* Name of the kernel the last FLOP pass ran (the pass picks one per matrix;
 * "" before the first pass). */
const char* spnnz_gpu_last_flop_kernel(spnnz_gpu_ctx* ctx);
/* The floor the FLOP pass's access pattern sets on the loaded matrices: the
 * same A.col loads (and, for gather_ms, the same uint16 degree gathers) with
 * none of the row logic, averaged over reps launches (ms, CUDA events).
 * bench.py reports the pass against it (roofline.pattern_ceiling_*). */
int spnnz_gpu_probe_flop_floor(spnnz_gpu_ctx* ctx, int reps, double* stream_ms, double* gather_ms);
/* Guard bands: with SPNNZ_GUARD=1 in the environment when the library
 * allocates, each device buffer is followed by 256 bytes of a known pattern,
 * checked when the buffer is freed and here for the live ones: reports how
 * many buffers were checked and how many bands changed (an out-of-bounds
 * write).  Synchronizes the device.  Test instrumentation. */
int spnnz_gpu_check_guards(int64_t* checked, int64_t* broken);
/* The context's CUDA stream (cudaStream_t), for callers that time on it. */
void* spnnz_gpu_stream(spnnz_gpu_ctx* ctx);
/* Ordering of DEVICE-residency inputs: every call that reads one first makes
 * the context's (non-blocking) stream wait for the work queued on `stream`
 * (a cudaStream_t) at the time of the call -- default NULL, the legacy
 * default stream.  A caller that produces its inputs on another stream
 * names it here (or synchronizes it before the call). */
int spnnz_gpu_set_input_stream(spnnz_gpu_ctx* ctx, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPNNZ_GPU_CAPI_H */
