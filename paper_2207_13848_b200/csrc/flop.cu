// Per-row FLOP profile (Algorithm 1): flop_i = sum_{j in A_i} |B_{A.col[j]}|.
// GPU restatement of spnnz::compute_flop (proj/include/spnnz/flop.hpp:25-60,
// hot loop :41-50), plus sampled_flop (:64-74).
//
// Decomposition: merge path over the sequence of M row-ends and nnz(A)
// nonzeros (Merrill & Garland, merge-based SpMV).  Each 256-thread block owns
// a tile of exactly 2048 items, so R-MAT hub rows (40 K nonzeros) and runs of
// empty rows balance perfectly.  Per tile:
//   0. (once per call) k_degree turns B.rpt into an int32 row-length array
//      (4 B per B row: 67 MB at config 5, L2-resident under an evict_last
//      policy, where the int64 pair B.rpt[k], B.rpt[k+1] (134 MB) is not);
//   1. coalesced, evict_first loads of A.col for the tile's nonzeros, and
//      for each one the gather deg[A.col[j]] (all 8 per thread issued back to
//      back), staged in shared memory;
//   2. every thread walks its 8 merge-path items out of shared memory; a
//      block-wide segmented scan over (row, partial) pairs joins rows that
//      cross thread boundaries (no shared-memory atomics: 64-bit ATOMS is a
//      CAS loop on sm_100 and serialises on hub rows);
//   3. rows that end in the tile are written once (coalesced); the partial
//      sum of the row still open at the tile's end is carried out and added by
//      k_flop_fixup, which also reduces F and the row maximum.
// Algorithmic bytes per launch: 8(M+1) A.rpt + 4 nnz A.col + 8(K+1) B.rpt
// + 8M flop written (the degree array's 4K write + re-reads are extra
// traffic, counted against us).  Integer-only: bit-exact.
#include <cub/block/block_scan.cuh>

#include "device_common.cuh"
#include "kernels.h"

namespace spnnz_gpu {
namespace {

// Merge-path search over a[0..a_len) (row ends) vs the counting sequence
// [0, b_len): returns the number of row-ends consumed at diagonal d.
template <typename LoadEnd>
__device__ __forceinline__ int64_t merge_search(int64_t d, int64_t a_len, int64_t b_len,
                                                LoadEnd end_at) {
    int64_t lo = d - b_len > 0 ? d - b_len : 0;
    int64_t hi = d < a_len ? d : a_len;
    while (lo < hi) {
        const int64_t pivot = (lo + hi) >> 1;
        if (end_at(pivot) <= d - pivot - 1)
            lo = pivot + 1;
        else
            hi = pivot;
    }
    return lo;
}

__global__ void k_degree(const int64_t* __restrict__ brpt, int64_t k_rows, int32_t* __restrict__ deg) {
    const uint64_t first = policy_evict_first(), last = policy_evict_last();
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < k_rows;
         k += int64_t(gridDim.x) * blockDim.x) {
        const long long lo = ld_stream_i64(reinterpret_cast<const long long*>(brpt) + k, first);
        const long long hi = ld_stream_i64(reinterpret_cast<const long long*>(brpt) + k + 1, first);
        st_keep_i32(deg + k, static_cast<int32_t>(hi - lo), last);
    }
}

__global__ void k_flop_partition(const int64_t* __restrict__ arpt, int32_t m, int64_t nnz,
                                 int64_t tiles, int32_t* __restrict__ tile_x) {
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (t > tiles) return;
    const int64_t total = int64_t(m) + nnz;
    const int64_t d = t * kFlopTile < total ? t * kFlopTile : total;
    const int64_t base = arpt[0];
    tile_x[t] = static_cast<int32_t>(
        merge_search(d, m, nnz, [&](int64_t i) { return __ldg(&arpt[i + 1]) - base; }));
}

// (row, partial sum) pairs for the block-wide reduce-by-row of carries.
struct RowCarry {
    int row;
    long long val;
};
struct RowCarryOp {
    __device__ __forceinline__ RowCarry operator()(const RowCarry& a, const RowCarry& b) const {
        return RowCarry{b.row, a.row == b.row ? a.val + b.val : b.val};
    }
};

// Shared-memory index with one pad word per 32: the merge-path walk reads
// item 8t+k in thread t, which would otherwise be an 8-way bank conflict.
__device__ __forceinline__ int pad(int i) { return i + (i >> 5); }

template <int BLOCK, int IPT>
__global__ void __launch_bounds__(BLOCK)
k_flop(const int64_t* __restrict__ arpt, const int32_t* __restrict__ acol,
       const int32_t* __restrict__ bdeg, int32_t m, int64_t nnz,
       const int32_t* __restrict__ tile_x, int64_t* __restrict__ flop,
       long long* __restrict__ tile_carry, long long* __restrict__ tile_total,
       long long* __restrict__ tile_max) {
    constexpr int TILE = BLOCK * IPT;
    constexpr int PADDED = TILE + TILE / 32 + 1;
    __shared__ int32_t s_end[PADDED];
    __shared__ int32_t s_deg[PADDED];
    __shared__ unsigned long long s_acc[TILE + 1];
    __shared__ long long s_red[BLOCK / 32];
    using BlockCarryScan = cub::BlockScan<RowCarry, BLOCK>;
    __shared__ typename BlockCarryScan::TempStorage s_scan;

    const uint64_t first = policy_evict_first(), last = policy_evict_last();
    const int64_t t = blockIdx.x;
    const int64_t base = __ldg(&arpt[0]);
    const int64_t total_items = int64_t(m) + nnz;
    const int64_t d0 = t * TILE;
    const int64_t d1 = d0 + TILE < total_items ? d0 + TILE : total_items;
    const int32_t x0 = tile_x[t], x1 = tile_x[t + 1];
    const int64_t y0 = d0 - x0, y1 = d1 - x1;
    const int nrows = x1 - x0;
    const int nz = static_cast<int>(y1 - y0);
    const int tid = threadIdx.x;

    for (int i = tid; i < nrows; i += BLOCK)
        s_end[pad(i)] = static_cast<int32_t>(
            ld_stream_i64(reinterpret_cast<const long long*>(arpt) + x0 + i + 1, first) - base - y0);

    // Column loads (coalesced, evict_first) then all degree gathers in flight.
    const int32_t* tcol = acol + base + y0;
    int32_t c[IPT];
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
        const int i = tid + k * BLOCK;
        c[k] = i < nz ? ld_stream_i32(tcol + i, first) : 0;
    }
    int32_t dg[IPT];
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
        const int i = tid + k * BLOCK;
        dg[k] = i < nz ? ld_keep_i32(bdeg + c[k], last) : 0;
    }
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
        const int i = tid + k * BLOCK;
        if (i < nz) s_deg[pad(i)] = dg[k];
    }
    __syncthreads();

    // Walk this thread's IPT merge-path items.  Rows ending inside the
    // thread's range after its first row-end are complete; the first one may
    // owe a carry from preceding threads, and the row still open at the end
    // is this thread's carry-out.  A block-wide segmented scan of the
    // (row, carry) pairs resolves both without shared-memory atomics.
    const int items = nrows + nz;
    const int td = tid * IPT < items ? tid * IPT : items;
    const int tend = td + IPT < items ? td + IPT : items;
    int x = static_cast<int>(
        merge_search(td, nrows, nz, [&](int64_t i) { return (int64_t)s_end[pad(static_cast<int>(i))]; }));
    int y = td - x;
    long long acc = 0, tsum = 0, first_val = 0;
    int first_row = -1;
    for (int k = td; k < tend; ++k) {
        if (x < nrows && s_end[pad(x)] <= y) {
            if (first_row < 0) {
                first_row = x;
                first_val = acc;
            } else {
                s_acc[x] = static_cast<unsigned long long>(acc);
            }
            acc = 0;
            ++x;
        } else {
            const long long dv = s_deg[pad(y)];
            acc += dv;
            tsum += dv;
            ++y;
        }
    }
    RowCarry mine{x, acc}, before;
    BlockCarryScan(s_scan).ExclusiveScan(mine, before, RowCarry{-1, 0}, RowCarryOp());
    if (first_row >= 0)
        s_acc[first_row] = static_cast<unsigned long long>(
            first_val + (before.row == first_row ? before.val : 0));
    if (tid == BLOCK - 1) {
        // carry-out of the tile: the open row's partial over the whole tile
        const RowCarry tot = RowCarryOp()(before, mine);
        s_acc[nrows] = static_cast<unsigned long long>(tot.row == nrows ? tot.val : 0);
    }
    __syncthreads();

    // Rows x0 .. x1-1 end in this tile.  Row x0 may have started in an
    // earlier tile (carry-in): its final value is known only after the fixup.
    const bool carry_in = nrows > 0 && (__ldg(&arpt[x0]) - base) < y0;
    long long tmax = 0;
    for (int i = tid; i < nrows; i += BLOCK) {
        const long long v = static_cast<long long>(s_acc[i]);
        flop[x0 + i] = v;
        if (!(i == 0 && carry_in)) tmax = v > tmax ? v : tmax;
    }
    const long long bsum = block_sum_ll<BLOCK>(tsum, s_red);
    const long long bmax = block_max_ll<BLOCK>(tmax, s_red);
    if (tid == 0) {
        tile_total[t] = bsum;
        tile_max[t] = bmax;
        tile_carry[t] = static_cast<long long>(s_acc[nrows]);
    }
}

// Adds carried partial sums to the rows that span tiles (one thread per first
// carrying tile of a row) and reduces F and max over all tiles.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
k_flop_fixup(const int32_t* __restrict__ tile_x, int64_t tiles, int32_t m,
             const long long* __restrict__ tile_carry, const long long* __restrict__ tile_total,
             const long long* __restrict__ tile_max, int64_t* __restrict__ flop,
             long long* __restrict__ totals) {
    __shared__ long long s_red[BLOCK / 32];
    const int64_t t = blockIdx.x * int64_t(BLOCK) + threadIdx.x;
    long long sum = 0, mx = 0;
    if (t < tiles) {
        sum = tile_total[t];
        mx = tile_max[t];
        const int32_t r = tile_x[t + 1];
        const bool first = (r < m) && (t == 0 || tile_x[t] != r);
        if (first) {
            long long carry = 0;
            for (int64_t u = t; u < tiles && tile_x[u + 1] == r; ++u) carry += tile_carry[u];
            const long long v = flop[r] + carry;
            flop[r] = v;
            mx = v > mx ? v : mx;
        }
    }
    sum = block_sum_ll<BLOCK>(sum, s_red);
    mx = block_max_ll<BLOCK>(mx, s_red);
    if (threadIdx.x == 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&totals[kF]),
                  static_cast<unsigned long long>(sum));
        atomicMax(reinterpret_cast<unsigned long long*>(&totals[kMax]),
                  static_cast<unsigned long long>(mx));
    }
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
k_sampled_flop(const int64_t* __restrict__ flop, int32_t row_lo, int32_t local_rows,
               const int32_t* __restrict__ rows, int64_t n, long long* __restrict__ totals) {
    __shared__ long long s_red[BLOCK / 32];
    long long s = 0;
    for (int64_t i = blockIdx.x * int64_t(BLOCK) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * BLOCK) {
        const int32_t r = rows[i] - row_lo;
        if (r >= 0 && r < local_rows) s += flop[r];
    }
    s = block_sum_ll<BLOCK>(s, s_red);
    if (threadIdx.x == 0 && s)
        atomicAdd(reinterpret_cast<unsigned long long*>(&totals[kFStar]),
                  static_cast<unsigned long long>(s));
}

__global__ void k_check_rows(const int32_t* __restrict__ rows, int64_t n, int32_t num_rows,
                             int32_t* bad) {
    const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (i < n && (rows[i] < 0 || rows[i] >= num_rows)) atomicAdd(bad, 1);
}

}  // namespace

cudaError_t launch_flop_partition(const DevCsr& a, const FlopScratch& s, cudaStream_t stream) {
    const int64_t tiles = flop_tiles(a);
    if (a.rows == 0) return cudaSuccess;
    const int block = 256;
    const int64_t grid = (tiles + 1 + block - 1) / block;
    k_flop_partition<<<static_cast<unsigned>(grid), block, 0, stream>>>(a.rpt, a.rows, a.nnz, tiles,
                                                                      s.tile_x);
    return cudaGetLastError();
}

cudaError_t launch_degree(const int64_t* brpt, int64_t k_rows, int32_t* deg, int num_sms,
                          cudaStream_t stream) {
    if (k_rows == 0) return cudaSuccess;
    int64_t grid = (k_rows + 255) / 256;
    if (grid > int64_t(num_sms) * 16) grid = int64_t(num_sms) * 16;
    k_degree<<<static_cast<unsigned>(grid), 256, 0, stream>>>(brpt, k_rows, deg);
    return cudaGetLastError();
}

cudaError_t launch_flop(const DevCsr& a, const int32_t* bdeg, const FlopScratch& s, int64_t* flop,
                        long long* totals, cudaStream_t stream) {
    const int64_t tiles = flop_tiles(a);
    if (tiles == 0) return cudaSuccess;
    k_flop<kFlopBlock, kFlopIpt><<<static_cast<unsigned>(tiles), kFlopBlock, 0, stream>>>(
        a.rpt, a.col, bdeg, a.rows, a.nnz, s.tile_x, flop, s.tile_carry, s.tile_total, s.tile_max);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    constexpr int FB = 256;
    k_flop_fixup<FB><<<static_cast<unsigned>((tiles + FB - 1) / FB), FB, 0, stream>>>(
        s.tile_x, tiles, a.rows, s.tile_carry, s.tile_total, s.tile_max, flop, totals);
    return cudaGetLastError();
}

cudaError_t launch_sampled_flop(const int64_t* flop, int32_t row_lo, int32_t local_rows,
                                const int32_t* rows, int64_t n, long long* totals,
                                cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    constexpr int B = 256;
    int64_t grid = (n + B - 1) / B;
    if (grid > 1024) grid = 1024;
    k_sampled_flop<B><<<static_cast<unsigned>(grid), B, 0, stream>>>(flop, row_lo, local_rows, rows,
                                                                    n, totals);
    return cudaGetLastError();
}

cudaError_t launch_check_rows(const int32_t* rows, int64_t n, int32_t num_rows, int32_t* bad,
                              cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    k_check_rows<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(rows, n, num_rows, bad);
    return cudaGetLastError();
}

}  // namespace spnnz_gpu
