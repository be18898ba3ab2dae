/* Host-side utilities of the B200 predictor (paper_2207_13848_b200/_lib/
 * libspnnz_gen.so): deterministic input generators and Matrix Market I/O.
 * Plain C ABI; matrices come back in malloc'd arrays released with
 * spnnz_gen_free.  These are the inputs of the corpus harness
 * (include/spnnz_gpu/harness.hpp), not part of the GPU path.
 */
#ifndef SPNNZ_GPU_HOST_H
#define SPNNZ_GPU_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t rows, cols;
    int64_t nnz;
    int64_t* rpt; /* rows + 1 */
    int32_t* col; /* nnz */
} spnnz_gen_csr;

void spnnz_gen_free(spnnz_gen_csr* m);

/* spnnz::generate_synthetic (synthetic.hpp:92-154); model 0 uniform,
 * 1 banded, 2 power-law.  0 ok, 3 infeasible spec (invalid_argument). */
int spnnz_gen_synthetic(int model, int32_t rows, int32_t cols, double target_nnz_per_row,
                        uint64_t seed, int32_t bandwidth, double skew, int threads,
                        spnnz_gen_csr* out);

/* spnnz::read_matrix_market (matrix_market.hpp:89-196), structure only.
 * 0 ok; 4 parse error: err holds the reference's message "<what> (line N)";
 * 5 I/O error; 6 out of memory. */
int spnnz_mm_read(const char* path, int threads, spnnz_gen_csr* out, char* err, int errcap);

/* spnnz::write_matrix_market (matrix_market.hpp:200-211): pattern, general. */
int spnnz_mm_write(const char* path, const spnnz_gen_csr* m);

#ifdef __cplusplus
}
#endif

#endif /* SPNNZ_GPU_HOST_H */
