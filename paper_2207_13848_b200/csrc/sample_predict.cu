// Seeded row sampler and the fused predict kernel.
//
// k_sample restates spnnz::make_sample_plan's draw loop
// (proj/include/spnnz/predict.hpp:48-54 over rng.hpp:14-24) one thread per
// draw: SplitMix64 is counter based (state_r = seed + (r+1)*gamma), so draw r
// needs no predecessor.  u = (z >> 11) * 2^-53 is exact; M * u is one IEEE
// multiply (round-to-nearest, __dmul_rn keeps the compiler from contracting)
// and the int32 cast truncates toward zero (__double2int_rz), with the
// reference's rid >= M guard.  Indices are therefore bit-identical.
//
// k_predict restates predict_row_structure / _ceil (predict.hpp:126-151):
// out = min(flop, (int64)ceil(flop / cr)) with an IEEE division (__ddiv_rn,
// never a reciprocal multiply), optional real view flop / cr.  When fed the
// device totals it first derives cr = f*/z* (or 1) exactly like
// collect_sample_stats / predict_proposed (predict.hpp:86-89, :111-117), so
// the whole pipeline runs without a host round trip.  Streaming: 16-byte
// loads of the profile, 16-byte evict-first stores.  8 B read + 8 B written
// per row (+8 B for the real view).
#include <atomic>

#include "device_common.cuh"
#include "kernels.h"

namespace spnnz_gpu {
namespace {

__global__ void k_sample(uint64_t seed, int32_t num_rows, int64_t n, int32_t* __restrict__ rows) {
    const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (r >= n) return;
    rows[r] = draw_row(seed, static_cast<uint64_t>(r), num_rows);
}

#ifndef SPNNZ_PRED_MINB
#define SPNNZ_PRED_MINB 6  // 40 registers: 1536 resident threads per SM
#endif
#ifndef SPNNZ_PRED_U
#define SPNNZ_PRED_U 4
#endif

// The IEEE quotient out of line: the reciprocal path below certifies almost
// every row, and keeping __ddiv_rn's slow path out of the kernel body keeps
// its register count (hence resident threads) low.
__device__ __noinline__ double div_slow(double a, double b) { return __ddiv_rn(a, b); }

// ceil_view (device_common.cuh) with the division through FastDiv: q is the
// correctly rounded f / cr either way.
__device__ __forceinline__ long long ceil_view_fast(long long f, const FastDiv& div, double* q_out) {
    if (f == 0) {
        *q_out = 0.0;
        return 0;
    }
    double q;
    if (!div.fast(static_cast<double>(f), &q)) q = div_slow(static_cast<double>(f), div.b);
    *q_out = q;
    return ceil_of(f, q);
}

template <bool CEIL, bool REAL>
__global__ void __launch_bounds__(256, SPNNZ_PRED_MINB)
k_predict(const int64_t* __restrict__ flop, int64_t m, const long long* __restrict__ totals,
          double cr_in, int64_t* __restrict__ ceil_out, double* __restrict__ real_out) {
    FastDiv div;
    div.init(totals ? predicted_cr(totals[kFStar], totals[kZStar]) : cr_in);

    const int64_t pairs = m >> 1;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(flop) |
                          (CEIL ? reinterpret_cast<uintptr_t>(ceil_out) : 0) |
                          (REAL ? reinterpret_cast<uintptr_t>(real_out) : 0)) & 15) == 0;
    if (vec_ok) {
        // kU pairs per thread per step, their loads issued back to back
        constexpr int kU = SPNNZ_PRED_U;
        const longlong2* f2 = reinterpret_cast<const longlong2*>(flop);
        for (int64_t i0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i0 < pairs; i0 += kU * stride) {
            longlong2 f[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int64_t i = i0 + u * stride;
                f[u] = i < pairs ? ld_stream_ll2(&f2[i]) : make_longlong2(0, 0);
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int64_t i = i0 + u * stride;
                if (i < pairs) {
                    double q0, q1;
                    const long long c0 = ceil_view_fast(f[u].x, div, &q0);
                    const long long c1 = ceil_view_fast(f[u].y, div, &q1);
                    if (CEIL) st_stream_ll2(reinterpret_cast<longlong2*>(ceil_out) + i, make_longlong2(c0, c1));
                    if (REAL) st_stream_d2(reinterpret_cast<double2*>(real_out) + i, make_double2(q0, q1));
                }
            }
        }
        if ((m & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
            double q;
            const long long c = ceil_view_fast(flop[m - 1], div, &q);
            if (CEIL) ceil_out[m - 1] = c;
            if (REAL) real_out[m - 1] = q;
        }
    } else {
        for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += stride) {
            double q;
            const long long c = ceil_view_fast(flop[i], div, &q);
            if (CEIL) ceil_out[i] = c;
            if (REAL) real_out[i] = q;
        }
    }
}

// One NCCL all-reduce for sums AND the max: every rank writes its slots
// [first, first + count) (and kMax) into its own row of a world x kTotals
// table that is zero elsewhere; a SUM all-reduce of the table gathers every
// rank's values, and k_totals_finish reduces the rows (sum, or max for kMax).
__global__ void k_totals_spread(const long long* __restrict__ totals, long long* __restrict__ table, int rank,
                                int world) {
    for (int i = threadIdx.x; i < world * kTotals; i += blockDim.x)
        table[i] = i / kTotals == rank ? totals[i % kTotals] : 0;
}

__global__ void k_totals_finish(long long* __restrict__ totals, const long long* __restrict__ table, int world,
                                int first, int count, int with_max) {
    const int i = threadIdx.x;
    if (i >= kTotals) return;
    const bool sum = i >= first && i < first + count;
    const bool mx = with_max && i == kMax;
    if (!sum && !mx) return;
    long long v = sum ? 0 : table[i];
    for (int r = 0; r < world; ++r) {
        const long long x = table[r * kTotals + i];
        v = sum ? v + x : (x > v ? x : v);
    }
    totals[i] = v;
}

}  // namespace

cudaError_t launch_totals_spread(const long long* totals, long long* table, int rank, int world,
                                 cudaStream_t stream) {
    k_totals_spread<<<1, 256, 0, stream>>>(totals, table, rank, world);
    return cudaGetLastError();
}

cudaError_t launch_totals_finish(long long* totals, const long long* table, int world, int first, int count,
                                 bool with_max, cudaStream_t stream) {
    k_totals_finish<<<1, 32, 0, stream>>>(totals, table, world, first, count, with_max ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_sample(uint64_t seed, int32_t num_rows, int64_t n, int32_t* rows,
                          cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    k_sample<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(seed, num_rows, n, rows);
    return cudaGetLastError();
}

cudaError_t launch_predict(const int64_t* flop, int64_t m, const long long* totals, double cr,
                           int64_t* ceil_out, double* real_out, int num_sms, cudaStream_t stream) {
    if (m == 0 || (!ceil_out && !real_out)) return cudaSuccess;
    // 32 blocks of 256 per SM (measured best of 4-32 x unroll 1-8 at
    // config 5: 0.068 ms, 60 % of the copy bandwidth), grid-stride over
    // 16-byte pairs.
    // one block per 256 threads x SPNNZ_PRED_U pairs, so a small shard (a
    // rank's rows at N = 8) runs as one wave with every load in flight
    // instead of several waves of one pair per thread (19 -> ~7 us at 2.7 M rows)
    int64_t grid = ((m >> 1) + 256 * SPNNZ_PRED_U - 1) / (256 * SPNNZ_PRED_U);
#ifndef SPNNZ_PRED_GRID
#define SPNNZ_PRED_GRID 32
#endif
    // at most one wave of resident blocks (a second, partial wave of a small
    // view doubled its time: 71 registers held 3 blocks per SM)
    static std::atomic<int> resident[3] = {0, 0, 0};
    const int kind = ceil_out && real_out ? 0 : ceil_out ? 1 : 2;
    int per_sm = resident[kind].load(std::memory_order_relaxed);
    if (per_sm == 0) {
        if (kind == 0)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_predict<true, true>, 256, 0);
        else if (kind == 1)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_predict<true, false>, 256, 0);
        else
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_predict<false, true>, 256, 0);
        if (per_sm < 1) per_sm = 1;
        resident[kind].store(per_sm, std::memory_order_relaxed);
    }
    int64_t cap = int64_t(num_sms) * per_sm;
    if (cap > int64_t(num_sms) * SPNNZ_PRED_GRID) cap = int64_t(num_sms) * SPNNZ_PRED_GRID;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    const unsigned g = static_cast<unsigned>(grid);
    if (ceil_out && real_out)
        k_predict<true, true><<<g, 256, 0, stream>>>(flop, m, totals, cr, ceil_out, real_out);
    else if (ceil_out)
        k_predict<true, false><<<g, 256, 0, stream>>>(flop, m, totals, cr, ceil_out, real_out);
    else
        k_predict<false, true><<<g, 256, 0, stream>>>(flop, m, totals, cr, ceil_out, real_out);
    return cudaGetLastError();
}

}  // namespace spnnz_gpu
