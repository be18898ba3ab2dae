// Per-row FLOP profile (Algorithm 1): flop_i = sum_{j in A_i} |B_{A.col[j]}|.
// GPU restatement of spnnz::compute_flop (proj/include/spnnz/flop.hpp:25-60,
// hot loop :41-50), plus sampled_flop (:64-74).  A pattern SpMV y = A * deg(B).
//
// Decomposition ("nnz tiles"): A's nonzeros are cut into fixed tiles of
// kFlopTile = 4096 entries aligned to absolute multiples of 4096, one
// 256-thread block per tile, so hub rows and runs of empty rows cost the
// same per entry.  A tile OWNS the rows that start inside it.  Per call:
//   0. k_degree turns B.rpt into a uint16 row-length array with an escape
//      value for rows of >= 65535 entries (2 B per B row: 34 MB at config 5,
//      L2-resident under an evict_last policy -- the int64 pair
//      B.rpt[k], B.rpt[k+1] is 134 MB and is not);
//   1. k_flop_partition: first owned row of every tile (lower_bound in rpt);
//   2. k_flop, per tile: 16-byte evict_first loads of the tile's A.col into
//      shared memory, then the deg[] gathers (8 per thread in flight, lanes
//      on consecutive entries), staged in shared memory; each thread then sums one owned row's slice of the staged
//      degrees (rows longer than 64 in the tile go to a warp each), writes
//      flop[row] and the tile's partials: F, max, and the leading segment
//      that belongs to a row owned by an earlier tile;
//   3. k_flop_fixup adds the leading segments to the long rows they continue
//      and reduces F and max over tiles.
// Per entry ~10 thread instructions (a merge-path walk cost ~90).
// Algorithmic bytes: 8(M+1) A.rpt + 4 nnz A.col + 8(K+1) B.rpt + 8M flop
// (the 2K-byte degree array's write and re-reads are extra traffic).
// Integer-only: bit-exact.
#include "device_common.cuh"
#include "kernels.h"

namespace spnnz_gpu {
namespace {

constexpr int kLongRow = 64;  // in-tile row slices longer than this go to a warp

// deg16[k] = min(B.rpt[k+1] - B.rpt[k], 0xFFFF); 0xFFFF means "look the
// exact length up in B.rpt" (rows with >= 65535 entries are rare).
__global__ void k_degree(const int64_t* __restrict__ brpt, int64_t k_rows,
                         uint16_t* __restrict__ deg) {
    const uint64_t first = policy_evict_first(), last = policy_evict_last();
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < k_rows;
         k += int64_t(gridDim.x) * blockDim.x) {
        const long long lo = ld_stream_i64(reinterpret_cast<const long long*>(brpt) + k, first);
        const long long hi = ld_stream_i64(reinterpret_cast<const long long*>(brpt) + k + 1, first);
        const long long d = hi - lo;
        st_keep_u16(deg + k, static_cast<uint16_t>(d < 0xFFFF ? d : 0xFFFF), last);
    }
}

__device__ __forceinline__ int64_t tile_start(int64_t base, int64_t nnz, int64_t t) {
    const int64_t s = (base / kFlopTile + t) * kFlopTile;
    return s > base ? (s < base + nnz ? s : base + nnz) : base;
}

// tile_row[t] = first row whose start offset is >= tile_start(t); the last
// tile also owns the trailing empty rows (tile_row[tiles] = m).
__global__ void k_flop_partition(const int64_t* __restrict__ arpt, int32_t m, int64_t base,
                                 int64_t nnz, int64_t tiles, int32_t* __restrict__ tile_row) {
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (t > tiles) return;
    if (t == tiles) {
        tile_row[t] = m;
        return;
    }
    const int64_t target = tile_start(base, nnz, t);
    int64_t lo = 0, hi = m;  // lower_bound over rpt[0..m]
    if (t == 0) hi = 0;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(&arpt[mid]) < target) lo = mid + 1; else hi = mid;
    }
    tile_row[t] = static_cast<int32_t>(lo);
}

template <int BLOCK, int V>
__global__ void __launch_bounds__(BLOCK, 5)
k_flop(const int64_t* __restrict__ arpt, const int32_t* __restrict__ acol,
       const uint16_t* __restrict__ bdeg, const int64_t* __restrict__ brpt, int32_t m,
       int64_t base, int64_t nnz, const int32_t* __restrict__ tile_row,
       int64_t* __restrict__ flop, long long* __restrict__ tile_lead,
       long long* __restrict__ tile_total, long long* __restrict__ tile_max) {
    constexpr int TILE = BLOCK * V;
    static_assert(TILE == kFlopTile, "tile size");
    __shared__ int32_t s_deg[TILE];
    __shared__ int32_t s_long_row[TILE / kLongRow + 2];
    __shared__ int32_t s_long_lo[TILE / kLongRow + 2];
    __shared__ int32_t s_long_hi[TILE / kLongRow + 2];
    __shared__ int s_nlong;
    __shared__ long long s_red[BLOCK / 32];

    const uint64_t first = policy_evict_first(), last = policy_evict_last();
    const int64_t t = blockIdx.x;
    const int64_t ts = tile_start(base, nnz, t), te = tile_start(base, nnz, t + 1);
    const int n = static_cast<int>(te - ts);
    const int tid = threadIdx.x;
    if (tid == 0) s_nlong = 0;

    // 1. stage the tile's degrees.  16-byte evict_first loads of A.col into
    //    shared memory (the tile start is a multiple of 4096 entries, so only
    //    a shard's first and last tiles are partial), then each thread reads
    //    entries tid, tid + 256, ... back (stride 1 across a warp, so the
    //    gathers of neighbouring entries share sectors when the columns are
    //    close, as in banded matrices), issues all its gathers, and stores
    //    the degrees in place.
    int32_t* s_col = s_deg;
    if (n == TILE && (reinterpret_cast<uintptr_t>(acol + ts) & 15) == 0) {
        const int4* src = reinterpret_cast<const int4*>(acol + ts);
        int4* dst = reinterpret_cast<int4*>(s_col);
#pragma unroll
        for (int k = 0; k < V / 4; ++k) dst[tid + k * BLOCK] = ld_stream_v4(src + tid + k * BLOCK, first);
    } else {
        for (int i = tid; i < n; i += BLOCK) s_col[i] = ld_stream_i32(acol + ts + i, first);
    }
    __syncthreads();
    long long tsum = 0;
#pragma unroll
    for (int h = 0; h < V; h += V / 2) {
        int32_t c[V / 2], dg[V / 2];
#pragma unroll
        for (int k = 0; k < V / 2; ++k) {
            const int i = tid + (h + k) * BLOCK;
            c[k] = i < n ? s_col[i] : 0;
        }
#pragma unroll
        for (int k = 0; k < V / 2; ++k) {
            const int i = tid + (h + k) * BLOCK;
            dg[k] = i < n ? static_cast<int32_t>(ld_keep_u16(bdeg + c[k], last)) : 0;
        }
#pragma unroll
        for (int k = 0; k < V / 2; ++k) {
            const int i = tid + (h + k) * BLOCK;
            if (i < n) {
                int32_t d = dg[k];
                if (d == 0xFFFF)
                    d = static_cast<int32_t>(__ldg(&brpt[c[k] + 1]) - __ldg(&brpt[c[k]]));
                s_deg[i] = d;
                tsum += d;
            }
        }
    }
    __syncthreads();

    // 2. owned rows [r0, r1): one thread per row, long slices deferred.
    const int32_t r0 = tile_row[t], r1 = tile_row[t + 1];
    long long tmax = 0;
    for (int32_t r = r0 + tid; r < r1; r += BLOCK) {
        const int64_t a = __ldg(&arpt[r]), b = __ldg(&arpt[r + 1]);
        const int lo = static_cast<int>(a - ts);
        const int hi = static_cast<int>((b < te ? b : te) - ts);
        if (hi - lo > kLongRow) {
            const int slot = atomicAdd(&s_nlong, 1);
            s_long_row[slot] = r;
            s_long_lo[slot] = lo;
            s_long_hi[slot] = hi;
        } else {
            long long sum = 0;
            for (int i = lo; i < hi; ++i) sum += s_deg[i];
            flop[r] = sum;
            if (b <= te) tmax = sum > tmax ? sum : tmax;  // complete within the tile
        }
    }
    // the leading slice [0, lead) continues row r0 - 1 from an earlier tile
    if (tid == 0) {
        const int64_t first_start = r0 < m ? __ldg(&arpt[r0]) : te;
        const int lead = static_cast<int>((first_start < te ? first_start : te) - ts);
        if (lead > 0) {
            const int slot = atomicAdd(&s_nlong, 1);
            s_long_row[slot] = -1;
            s_long_lo[slot] = 0;
            s_long_hi[slot] = lead;
        } else {
            tile_lead[t] = 0;
        }
    }
    __syncthreads();

    // 3. long slices: one warp each
    const int lane = tid & 31, warp = tid >> 5;
    for (int j = warp; j < s_nlong; j += BLOCK / 32) {
        long long sum = 0;
        for (int i = s_long_lo[j] + lane; i < s_long_hi[j]; i += 32) sum += s_deg[i];
        sum = warp_sum_ll(sum);
        if (lane == 0) {
            const int32_t r = s_long_row[j];
            if (r < 0) {
                tile_lead[t] = sum;
            } else {
                flop[r] = sum;
                if (__ldg(&arpt[r + 1]) <= te) tmax = sum > tmax ? sum : tmax;
            }
        }
    }
    const long long bsum = block_sum_ll<BLOCK>(tsum, s_red);
    const long long bmax = block_max_ll<BLOCK>(tmax, s_red);
    if (tid == 0) {
        tile_total[t] = bsum;
        tile_max[t] = bmax;
    }
}

// Adds each tile's leading slice to the row it continues (one thread per
// first continuing tile of a row, summing the run of tiles that continue the
// same row) and reduces F and max over all tiles.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK)
k_flop_fixup(const int32_t* __restrict__ tile_row, int64_t tiles,
             const long long* __restrict__ tile_lead, const long long* __restrict__ tile_total,
             const long long* __restrict__ tile_max, int64_t* __restrict__ flop,
             long long* __restrict__ totals) {
    __shared__ long long s_red[BLOCK / 32];
    const int64_t t = blockIdx.x * int64_t(BLOCK) + threadIdx.x;
    long long sum = 0, mx = 0;
    if (t < tiles) {
        sum = tile_total[t];
        mx = tile_max[t];
        // tile t continues row r = tile_row[t] - 1 when its leading slice is
        // non-empty; tile t is the first such tile unless tile t-1 owned no
        // row either (tile_row[t-1] == tile_row[t]).
        const int32_t r = tile_row[t] - 1;
        const bool first = t > 0 && r >= 0 && tile_row[t - 1] != tile_row[t];
        if (first) {
            long long carry = 0;
            for (int64_t u = t; u < tiles && tile_row[u] == r + 1; ++u) carry += tile_lead[u];
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

// Row-sortedness of B (the CsrMatrix invariant, csr.hpp:16-18), checked once
// at load: every descent col[j] < col[j-1] must sit at the start of a
// non-empty row.  cnt[0] += descents over all j, cnt[1] += descents at row
// starts; B is sorted iff they are equal.
__global__ void k_descents(const int32_t* __restrict__ col, int64_t nnz, unsigned long long* cnt) {
    unsigned long long d = 0;
    for (int64_t j = 1 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < nnz;
         j += int64_t(gridDim.x) * blockDim.x)
        d += __ldg(&col[j]) < __ldg(&col[j - 1]);
    d = warp_sum_ll(static_cast<long long>(d));
    if ((threadIdx.x & 31) == 0 && d) atomicAdd(&cnt[0], d);
}

__global__ void k_start_descents(const int64_t* __restrict__ rpt, const int32_t* __restrict__ col,
                                 int32_t rows, unsigned long long* cnt) {
    unsigned long long d = 0;
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < rows;
         r += int64_t(gridDim.x) * blockDim.x) {
        const int64_t j = rpt[r];
        if (j >= 1 && j < rpt[r + 1]) d += __ldg(&col[j]) < __ldg(&col[j - 1]);
    }
    d = warp_sum_ll(static_cast<long long>(d));
    if ((threadIdx.x & 31) == 0 && d) atomicAdd(&cnt[1], d);
}

}  // namespace

cudaError_t launch_check_sorted(const int64_t* rpt, const int32_t* col, int32_t rows, int64_t nnz,
                                unsigned long long* cnt, int num_sms, cudaStream_t stream) {
    cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), stream);
    const unsigned grid = static_cast<unsigned>(num_sms) * 8;
    if (nnz > 1) k_descents<<<grid, 256, 0, stream>>>(col, nnz, cnt);
    if (rows > 0) k_start_descents<<<grid, 256, 0, stream>>>(rpt, col, rows, cnt);
    return cudaGetLastError();
}

int64_t flop_tiles(const DevCsr& a) {
    if (a.rows == 0) return 0;
    if (a.nnz == 0) return 1;
    const int64_t end = a.base + a.nnz;
    return (end + kFlopTile - 1) / kFlopTile - a.base / kFlopTile;
}

cudaError_t launch_degree(const int64_t* brpt, int64_t k_rows, uint16_t* deg, int num_sms,
                          cudaStream_t stream) {
    if (k_rows == 0) return cudaSuccess;
    int64_t grid = (k_rows + 255) / 256;
    if (grid > int64_t(num_sms) * 16) grid = int64_t(num_sms) * 16;
    k_degree<<<static_cast<unsigned>(grid), 256, 0, stream>>>(brpt, k_rows, deg);
    return cudaGetLastError();
}

cudaError_t launch_flop_partition(const DevCsr& a, const FlopScratch& s, cudaStream_t stream) {
    const int64_t tiles = flop_tiles(a);
    if (tiles == 0) return cudaSuccess;
    const int block = 256;
    const int64_t grid = (tiles + 1 + block - 1) / block;
    k_flop_partition<<<static_cast<unsigned>(grid), block, 0, stream>>>(a.rpt, a.rows, a.base,
                                                                      a.nnz, tiles, s.tile_x);
    return cudaGetLastError();
}

cudaError_t launch_flop(const DevCsr& a, const uint16_t* bdeg, const int64_t* brpt,
                        const FlopScratch& s, int64_t* flop, long long* totals,
                        cudaStream_t stream) {
    const int64_t tiles = flop_tiles(a);
    if (tiles == 0) return cudaSuccess;
    k_flop<kFlopBlock, kFlopIpt><<<static_cast<unsigned>(tiles), kFlopBlock, 0, stream>>>(
        a.rpt, a.col, bdeg, brpt, a.rows, a.base, a.nnz, s.tile_x, flop, s.tile_carry,
        s.tile_total, s.tile_max);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    constexpr int FB = 256;
    k_flop_fixup<FB><<<static_cast<unsigned>((tiles + FB - 1) / FB), FB, 0, stream>>>(
        s.tile_x, tiles, s.tile_carry, s.tile_total, s.tile_max, flop, totals);
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
