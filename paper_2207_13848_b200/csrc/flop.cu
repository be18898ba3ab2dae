// Per-row FLOP profile (Algorithm 1): flop_i = sum_{j in A_i} |B_{A.col[j]}|.
// GPU restatement of spnnz::compute_flop (proj/include/spnnz/flop.hpp:25-60,
// hot loop :41-50), plus sampled_flop (:64-74).  A pattern SpMV y = A * deg(B).
//
// Decomposition ("nnz tiles"): A's nonzeros are cut into fixed tiles of
// kFlopTile = 2048 entries aligned to absolute multiples of 2048, one
// 128-thread block per tile (10 resident per SM; 128 measured 3 % faster
// than 256- and 64-thread tiles at configs 3 and 5), so hub rows and runs of
// empty rows cost the same per entry.  A tile OWNS the rows that start inside it.  Per call:
//   0. k_degree turns B.rpt into a uint16 row-length array with an escape
//      value for rows of >= 65535 entries (2 B per B row: 34 MB at config 5,
//      L2-resident under an evict_last policy -- the int64 pair
//      B.rpt[k], B.rpt[k+1] is 134 MB and is not);
//   1. the tile partition (first owned row of every tile): each A row marks
//      the tiles whose start falls inside it -- in the same pass over B.rpt
//      when A.rpt is a view of it (C = A*A), else k_tile_rows over A.rpt;
//   2. k_flop, per tile: each thread loads V = 16 consecutive A.col entries
//      (16-byte evict_first loads) and issues their 16 degree gathers at once
//      (evict_last); the tile's owned rows mark their starts in a tile-sized
//      shared bitmap; each thread sums its entries segment by segment in
//      registers (rows inside the thread are written directly) and a
//      block-wide segmented scan of (flag, partial, row) carries finishes the
//      rows that span threads.  Partials out: F, max, and the leading segment
//      that belongs to a row owned by an earlier tile;
//   3. k_flop_fixup adds the leading segments to the long rows they continue
//      and reduces F and max over tiles.
// No shared-memory round trip per entry: the L1/shared pipe is left to the
// gathers, which bound the pass (~1 L2 request per entry; at config 5 the pass
// runs at 86-89 % of the same loads with no row logic,
// tools/microbench/flop_ceiling.cu).
// Also here: the FLOP of listed rows straight from A and B.rpt (a flat
// decomposition into 128-entry chunks: the sampled rows' FLOP the symbolic
// binning and the multi-GPU split use) and the FLOP-balanced window of a
// sample list a rank counts (k_flop_window).
// Algorithmic bytes: 8(M+1) A.rpt + 4 nnz A.col + 8(K+1) B.rpt + 8M flop
// (the 2K-byte degree array's write and re-reads are extra traffic).
// Integer-only: bit-exact.
#include <atomic>
#include <type_traits>

#include <cub/block/block_scan.cuh>

#include "device_common.cuh"
#include "kernels.h"

namespace spnnz_gpu {
namespace {

__device__ __forceinline__ int64_t tile_start(int64_t base, int64_t nnz, int64_t t) {
    const int64_t s = (base / kFlopTile + t) * kFlopTile;
    return s > base ? (s < base + nnz ? s : base + nnz) : base;
}

// Tile partition by streaming (one A row per thread instead of one binary
// search per tile): tile_row[t] = first row r with rpt[r] >= tile_start(t),
// i.e. row r >= 1 is the answer for the tiles whose start lies in
// (rpt[r-1], rpt[r]].  For 1 <= t < tiles, tile_start(t) = (base/T + t) T
// exactly, so those tiles are t in [rpt[r-1]/T + 1, rpt[r]/T] - base/T.
// tile_row[0] = 0 and tile_row[tiles] = m are written by the caller's thread 0.
struct TileMarks {
    int32_t* tile_row = nullptr;  // null: no marking
    int64_t a_off = 0;            // A row r is B row a_off + r (A.rpt is a view of B.rpt)
    int32_t m = 0;
    int64_t base = 0, tiles = 0;
    // rows crossing no tile boundary (most) cost one shift-compare
    __device__ __forceinline__ void row(int32_t r, long long lo, long long hi) const {
        constexpr int kShift = __builtin_ctz(kFlopTile);
        const uint64_t q0 = static_cast<uint64_t>(lo) >> kShift, q1 = static_cast<uint64_t>(hi) >> kShift;
        if (q0 == q1) return;
        const int64_t b0 = static_cast<int64_t>(static_cast<uint64_t>(base) >> kShift);
        int64_t t0 = static_cast<int64_t>(q0) + 1 - b0, t1 = static_cast<int64_t>(q1) - b0;
        if (t0 < 1) t0 = 1;
        if (t1 > tiles - 1) t1 = tiles - 1;
        for (int64_t t = t0; t <= t1; ++t) tile_row[t] = r;
    }
    __device__ __forceinline__ void ends() const {
        tile_row[0] = 0;
        tile_row[tiles] = m;
    }
};

// deg16[k] = min(B.rpt[k+1] - B.rpt[k], 0xFFFF); 0xFFFF means "look the
// exact length up in B.rpt" (rows with >= 65535 entries are rare).  With
// marks on (C = A*A: A's row pointers are a view of B's), the same pass over
// B.rpt also writes A's tile partition.
__device__ __forceinline__ void degree_row(const TileMarks& mk, uint16_t* deg, int64_t k, long long lo,
                                           long long hi) {
    const long long d = hi - lo;
    deg[k] = static_cast<uint16_t>(d < 0xFFFF ? d : 0xFFFF);
    if (mk.tile_row && d > 0) {
        const int64_t r = k + 1 - mk.a_off;  // A row whose start is B.rpt[k + 1]
        if (r >= 1 && r <= mk.m) mk.row(static_cast<int32_t>(r), lo, hi);
    }
}

// Four rows per thread per step: B.rpt[k .. k+4] as two 16-byte loads plus
// one 8-byte load, all issued before any store, then one 8-byte store of the
// four degrees (the marking branch would otherwise serialise the loads).
__global__ void k_degree(const int64_t* __restrict__ brpt, int64_t k_rows,
                         uint16_t* __restrict__ deg, TileMarks mk, unsigned* __restrict__ escapes) {
    bool esc = false;  // a B row of >= 65535 entries (its degree escapes to B.rpt)
    const uint64_t first = policy_evict_first(), last = policy_evict_last();
    if (mk.tile_row && blockIdx.x == 0 && threadIdx.x == 0) mk.ends();
    const int64_t groups = k_rows >> 2;
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < groups;
         g += int64_t(gridDim.x) * blockDim.x) {
        const int64_t k = g << 2;
        const int4 v0 = ld_stream_v4(reinterpret_cast<const int4*>(brpt + k), first);
        const int4 v1 = ld_stream_v4(reinterpret_cast<const int4*>(brpt + k + 2), first);
        const long long r4 = ld_stream_i64(reinterpret_cast<const long long*>(brpt) + k + 4, first);
        long long r[5];
        r[0] = (static_cast<long long>(static_cast<unsigned>(v0.y)) << 32) | static_cast<unsigned>(v0.x);
        r[1] = (static_cast<long long>(static_cast<unsigned>(v0.w)) << 32) | static_cast<unsigned>(v0.z);
        r[2] = (static_cast<long long>(static_cast<unsigned>(v1.y)) << 32) | static_cast<unsigned>(v1.x);
        r[3] = (static_cast<long long>(static_cast<unsigned>(v1.w)) << 32) | static_cast<unsigned>(v1.z);
        r[4] = r4;
        uint64_t packed = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long d = r[j + 1] - r[j];
            packed |= static_cast<uint64_t>(d < 0xFFFF ? d : 0xFFFF) << (16 * j);
            esc |= d >= 0xFFFF;
        }
        asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(deg + k), "l"(packed), "l"(last));
        if (mk.tile_row) {
            // a row marks tiles only when it crosses a tile boundary: one
            // compare of the tile indices of its ends (equal for empty rows)
            constexpr int kShift = __builtin_ctz(kFlopTile);
            uint64_t q[5];
#pragma unroll
            for (int j = 0; j < 5; ++j) q[j] = static_cast<uint64_t>(r[j]) >> kShift;
            if (q[0] != q[4]) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int64_t row = k + j + 1 - mk.a_off;
                    if (q[j] != q[j + 1] && row >= 1 && row <= mk.m)
                        mk.row(static_cast<int32_t>(row), r[j], r[j + 1]);
                }
            }
        }
    }
    // the k_rows % 4 tail
    const int64_t t = (groups << 2) + blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (t < k_rows) {
        const long long lo = __ldg(&brpt[t]), hi = __ldg(&brpt[t + 1]);
        degree_row(mk, deg, t, lo, hi);
        esc |= hi - lo >= 0xFFFF;
    }
    if (escapes && __any_sync(0xffffffffu, esc) && (threadIdx.x & 31) == 0) atomicOr(escapes, 1u);
}

__global__ void k_tile_rows(const int64_t* __restrict__ arpt, TileMarks mk) {
    if (blockIdx.x == 0 && threadIdx.x == 0) mk.ends();
    for (int64_t r = 1 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r <= mk.m;
         r += int64_t(gridDim.x) * blockDim.x) {
        const long long lo = __ldg(&arpt[r - 1]), hi = __ldg(&arpt[r]);
        if (hi > lo) mk.row(static_cast<int32_t>(r), lo, hi);
    }
}

#ifdef SPNNZ_BINARY_PARTITION  // A/B reference: one binary search per tile
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
#endif

#ifndef SPNNZ_FLOP_MINB  // resident threads per SM the register budget targets
#define SPNNZ_FLOP_MINB 1280
#endif

#ifndef SPNNZ_FLOP_GATHER
#define SPNNZ_FLOP_GATHER 0
#endif
// The degree gather (A/B-tested variants: 0 evict_last hint, 1 plain __ldg,
// 2 evict_last without L1 allocation, 3 plain coherent load).
__device__ __forceinline__ uint16_t gather_deg(const uint16_t* p, uint64_t last) {
#if SPNNZ_FLOP_GATHER == 1
    return __ldg(p);
#elif SPNNZ_FLOP_GATHER == 2
    unsigned short v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(last));
    return v;
#elif SPNNZ_FLOP_GATHER == 3
    return *p;
#else
    return ld_keep_u16(p, last);
#endif
}

#ifndef SPNNZ_FLOP_COLLOAD
#define SPNNZ_FLOP_COLLOAD 3
#endif
// A.col loads: a thread's four 16-byte loads cover 64 contiguous bytes, 64 B
// apart across lanes, so two loads share each 32-byte sector.  Allocating in
// L1 (variant 1, the default; L2 still evict_first) lets the second load of a
// sector merge with the first: -2.4 % FLOP-pass time at config 5 versus the
// no-allocate load (0), as the pass is bound by L2 requests.
__device__ __forceinline__ int4 load_cols(const int4* p, uint64_t first) {
#if SPNNZ_FLOP_COLLOAD == 1
    int4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(first));
    return v;
#elif SPNNZ_FLOP_COLLOAD == 2
    return __ldg(p);
#else
    return ld_stream_v4(p, first);
#endif
}

// Segmented-sum carry across threads: (has a row start, carried value, row).
struct Carry {
    int flag;
    long long v;
    int32_t row;
};

__device__ __forceinline__ Carry carry_op(const Carry& a, const Carry& b) {
    Carry r;
    r.flag = a.flag | b.flag;
    r.v = b.flag ? b.v : a.v + b.v;
    r.row = b.flag ? b.row : a.row;
    return r;
}

__device__ __forceinline__ Carry shfl_up_carry(const Carry& c, int d) {
    Carry r;
    r.flag = __shfl_up_sync(0xffffffffu, c.flag, d);
    r.v = __shfl_up_sync(0xffffffffu, c.v, d);
    r.row = __shfl_up_sync(0xffffffffu, c.row, d);
    return r;
}

// The per-row prediction of a final flop value (fused predict).
struct Emit {
    FastDiv div;
    PredOut p;
    __device__ __forceinline__ void operator()(int32_t r, long long v) const {
        double q = 0.0;  // 0 / cr = +0 (cr >= 1)
        if (v == 0 || div.fast(static_cast<double>(v), &q)) {
            if (p.ceil) p.ceil[r] = ceil_of(v, q);
            if (p.real) p.real[r] = q;
        } else {
            const unsigned long long k = atomicAdd(p.nredo, 1ULL);
            if (k < static_cast<unsigned long long>(p.redo_cap)) p.redo[k] = r;
        }
    }
};

__device__ __forceinline__ Emit make_emit(const PredOut& p) {
    Emit e;
    e.div.init(p.on() ? predicted_cr(p.totals[kFStar], p.totals[kZStar]) : 1.0);
    e.p = p;
    return e;
}

// Degree sources: the uint16 degree array in global memory (L2-resident,
// gathered under evict_last) or a copy of it in shared memory (B with few
// rows: config 4's 65536 rows are a 128 KB table).  0xFFFF escapes to B.rpt.
// NOL1: a table far larger than L1 (config 5: 32 MB): gathers skip L1
// allocation (a compile-time choice: a runtime branch around the 16 gathers
// cost 5 % at config 5)
template <bool NOL1 = false>
struct GlobalDeg {
    const uint16_t* deg;
    uint64_t last;
    __device__ __forceinline__ int32_t operator()(int32_t c) const {
        if (NOL1) {
            unsigned short v;
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;"
                         : "=h"(v) : "l"(deg + c), "l"(last));
            return v;
        }
        return gather_deg(deg + c, last);
    }
};
struct SharedDeg {
    const uint16_t* deg;  // shared window
    __device__ __forceinline__ int32_t operator()(int32_t c) const { return deg[c]; }
};

// Barrier over the threads that work on one tile: the whole block, or one
// 128-thread group of a persistent block (named barrier 1 + group).
struct BlockBar {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
template <int THREADS>
struct GroupBar {
    int id;
    __device__ __forceinline__ void operator()() const {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(THREADS) : "memory");
    }
};

// Shared memory of one tile.
template <int BLOCK, int V>
struct TileSmem {
    static constexpr int TILE = BLOCK * V, NW = BLOCK / 32;
    uint32_t start[TILE / 32];  // bit i: an owned non-empty row starts at entry i
    int32_t rowat[TILE];        // ... and its id (read only where the bit is set); row mode: the tile's columns
    Carry wc[NW];
    long long red[NW], red2[NW];
};

struct TileArgs {
    const int64_t* __restrict__ arpt;
    const int32_t* __restrict__ acol;
    const int64_t* __restrict__ brpt;
    int64_t base, nnz;
    const int32_t* __restrict__ tile_row;
    int64_t* __restrict__ flop;
    long long* __restrict__ tile_lead;
    long long* __restrict__ tile_total;
    long long* __restrict__ tile_max;
    int prefetch_ahead;  // k_flop: L2-prefetch the columns of tile t + this (0: off)
};

// The exact degree of B row c given its uint16 entry (0xFFFF: look it up).
__device__ __forceinline__ int32_t exact_deg(int32_t d, int32_t c, const int64_t* brpt) {
    return d == 0xFFFF ? static_cast<int32_t>(__ldg(&brpt[c + 1]) - __ldg(&brpt[c])) : d;
}

// Tile totals: F and max in one pass (warp reductions, one shared slot pair
// per warp, warp 0 finishes both).
template <int BLOCK, int V, class Bar>
__device__ __forceinline__ void tile_totals(TileSmem<BLOCK, V>& sm, const TileArgs& g, int64_t t, int tid,
                                            long long tsum, long long tmax, Bar bar) {
    constexpr int NW = BLOCK / 32;
    const int lane = tid & 31, warp = tid >> 5;
    tsum = warp_sum_ll(tsum);
    tmax = warp_max_ll(tmax);
    if (lane == 0) {
        sm.red[warp] = tsum;
        sm.red2[warp] = tmax;
    }
    bar();
    if (warp == 0) {
        long long a = lane < NW ? sm.red[lane] : 0, b = lane < NW ? sm.red2[lane] : 0;
        a = warp_sum_ll(a);
        b = warp_max_ll(b);
        if (lane == 0) {
            g.tile_total[t] = a;
            g.tile_max[t] = b;
        }
    }
}

// L2 prefetch of a later tile's columns (one bulk-prefetch instruction: the
// tile is 8 KB, 16-byte aligned except at a shard's ends), so its col loads
// find them in L2 instead of waiting on HBM.
__device__ __forceinline__ void prefetch_tile(const TileArgs& g, int64_t t) {
    const int64_t ts = tile_start(g.base, g.nnz, t), te = tile_start(g.base, g.nnz, t + 1);
    const uintptr_t p0 = (reinterpret_cast<uintptr_t>(g.acol + ts) + 15) & ~uintptr_t(15);
    const uintptr_t p1 = reinterpret_cast<uintptr_t>(g.acol + te) & ~uintptr_t(15);
    if (p1 > p0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p0), "r"(static_cast<unsigned>(p1 - p0))
                     : "memory");
}

// Row mode, for banded A (27-point stencil: consecutive rows reach
// consecutive columns): the tile's columns are staged in shared memory
// (coalesced, conflict-free: thread tid loads entries tid + k BLOCK) and each
// thread walks whole rows, so a warp's k-th gathers hit ~32 consecutive
// degrees (one or two L1 lines) instead of ~9 clusters per instruction.  A
// row's gathers are issued 16 at a time (a stencil row is 27 entries: two
// rounds of loads in flight).
template <int BLOCK, int V, bool PRED, class Deg, class Bar>
__device__ __forceinline__ void flop_tile_rows(TileSmem<BLOCK, V>& sm, const TileArgs& g, int64_t t, int tid,
                                               int64_t ts, int n, int32_t r0, int32_t r1, Deg deg, Bar bar,
                                               const Emit& emit) {
    constexpr int W = 16;
    const uint64_t first = policy_evict_first();
    int64_t ra = 0, rb = 0;
    if (r0 + tid < r1) {
        ra = __ldg(&g.arpt[r0 + tid]);
        rb = __ldg(&g.arpt[r0 + tid + 1]);
    }
    const int64_t a0 = __ldg(&g.arpt[r0]);
    if (n == V * BLOCK && (reinterpret_cast<uintptr_t>(g.acol + ts) & 15) == 0) {
        // whole aligned tile: asynchronous 16-byte copies straight into shared
        // memory (chunk tid + k BLOCK: consecutive lanes, consecutive chunks)
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(sm.rowat));
#pragma unroll
        for (int k = 0; k < V / 4; ++k) {
            const int j = tid + k * BLOCK;
            asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst + 16 * j),
                         "l"(g.acol + ts + 4 * j), "l"(first)
                         : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    } else {
        int32_t c[V];
#pragma unroll
        for (int k = 0; k < V; ++k) {
            const int i = tid + k * BLOCK;
            c[k] = i < n ? ld_stream_i32(g.acol + ts + i, first) : 0;
        }
#pragma unroll
        for (int k = 0; k < V; ++k)
            if (tid + k * BLOCK < n) sm.rowat[tid + k * BLOCK] = c[k];
    }
    bar();
    const int64_t te = ts + n;
    long long tsum = 0, tmax = 0;
    // the leading slice (a row owned by an earlier tile): warp 0
    if (tid < 32) {
        const int lead_n = static_cast<int>((a0 < te ? a0 : te) - ts);
        long long s = 0;
        for (int i = tid; i < lead_n; i += 32) s += exact_deg(deg(sm.rowat[i]), sm.rowat[i], g.brpt);
        s = warp_sum_ll(s);
        if (tid == 0) {
            g.tile_lead[t] = s;
            tsum += s;
        }
    }
    for (int32_t r = r0 + tid; r < r1; r += BLOCK) {
        if (r != r0 + tid) {
            ra = __ldg(&g.arpt[r]);
            rb = __ldg(&g.arpt[r + 1]);
        }
        const int e0 = static_cast<int>(ra - ts), e1 = static_cast<int>((rb < te ? rb : te) - ts);
        long long s = 0;
        for (int e = e0; e < e1; e += W) {
            int32_t cc[W], d[W];
#pragma unroll
            for (int k = 0; k < W; ++k) cc[k] = e + k < e1 ? sm.rowat[e + k] : -1;
#pragma unroll
            for (int k = 0; k < W; ++k) d[k] = cc[k] >= 0 ? deg(cc[k]) : 0;
#pragma unroll
            for (int k = 0; k < W; ++k) s += cc[k] >= 0 ? exact_deg(d[k], cc[k], g.brpt) : 0;
        }
        tsum += s;
        g.flop[r] = s;  // partial when the row runs past the tile: the fixup adds the rest
        if (rb <= te) {
            tmax = s > tmax ? s : tmax;
            if (PRED) emit(r, s);
        }
    }
    tile_totals<BLOCK, V>(sm, g, t, tid, tsum, tmax, bar);
}

// One tile of kFlopTile entries by BLOCK threads (tid in [0, BLOCK)); ROWS:
// the row-mode instantiation (banded A, chosen on the host at load).
template <int BLOCK, int V, bool PRED, bool ROWS, class Deg, class Bar>
__device__ __forceinline__ void flop_tile(TileSmem<BLOCK, V>& sm, const TileArgs& g, int64_t t, int tid,
                                          Deg deg, Bar bar, const Emit& emit) {
    constexpr int TILE = BLOCK * V, NW = BLOCK / 32;
    static_assert(TILE == kFlopTile && (V == 8 || V == 16 || V == 32), "tile size");
    const uint64_t first = policy_evict_first();
    const int64_t ts = tile_start(g.base, g.nnz, t), te = tile_start(g.base, g.nnz, t + 1);
    const int n = static_cast<int>(te - ts);
    const int lane = tid & 31, warp = tid >> 5;
    if (ROWS) {  // row mode: owned rows averaging <= 48 entries in a banded matrix
        const int32_t q0 = g.tile_row[t], q1 = g.tile_row[t + 1];
        if (q1 > q0 && n <= 48 * (q1 - q0)) {
            flop_tile_rows<BLOCK, V, PRED>(sm, g, t, tid, ts, n, q0, q1, deg, bar, emit);
            return;
        }
    }
    for (int k = tid; k < TILE / 32; k += BLOCK) sm.start[k] = 0u;

    // 1. this thread's V consecutive entries: columns (16-byte evict_first
    //    loads when the tile is whole)
    const int i0 = tid * V;
    int32_t c[V];
#if SPNNZ_FLOP_COLLOAD == 3
    // 32-byte loads (sm_100 LDG.256): a thread's load is one whole sector, so
    // the columns need no L1 merging and skip L1 (left to the degree lines)
    if (n == TILE && (reinterpret_cast<uintptr_t>(g.acol + ts) & 31) == 0) {
        const int32_t* src = g.acol + ts + i0;
#pragma unroll
        for (int k = 0; k < V / 8; ++k)
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                         : "=r"(c[8 * k]), "=r"(c[8 * k + 1]), "=r"(c[8 * k + 2]), "=r"(c[8 * k + 3]),
                           "=r"(c[8 * k + 4]), "=r"(c[8 * k + 5]), "=r"(c[8 * k + 6]), "=r"(c[8 * k + 7])
                         : "l"(src + 8 * k), "l"(first));
    } else
#endif
    if (n == TILE && (reinterpret_cast<uintptr_t>(g.acol + ts) & 15) == 0) {
        const int4* src = reinterpret_cast<const int4*>(g.acol + ts + i0);
#pragma unroll
        for (int k = 0; k < V / 4; ++k) {
            const int4 x = load_cols(src + k, first);
            c[4 * k] = x.x;
            c[4 * k + 1] = x.y;
            c[4 * k + 2] = x.z;
            c[4 * k + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < V; ++k) c[k] = i0 + k < n ? ld_stream_i32(g.acol + ts + i0 + k, first) : -1;
    }
    //    ... then all V degree gathers in flight
    int32_t d[V];
#pragma unroll
    for (int k = 0; k < V; ++k) d[k] = c[k] >= 0 ? deg(c[k]) : 0;
#pragma unroll
    for (int k = 0; k < V; ++k)
        if (d[k] == 0xFFFF) d[k] = static_cast<int32_t>(__ldg(&g.brpt[c[k] + 1]) - __ldg(&g.brpt[c[k]]));
    long long tsum = 0;
#pragma unroll
    for (int k = 0; k < V; ++k) tsum += d[k];
    bar();  // the start bitmap is clear

    // 2. owned rows [r0, r1): mark where the non-empty ones start; empty ones are 0
    const int32_t r0 = g.tile_row[t], r1 = g.tile_row[t + 1];
    for (int32_t r = r0 + tid; r < r1; r += BLOCK) {
        const int64_t ra = __ldg(&g.arpt[r]), rb = __ldg(&g.arpt[r + 1]);
        if (rb > ra) {
            const int pos = static_cast<int>(ra - ts);
            atomicOr(&sm.start[pos >> 5], 1u << (pos & 31));
            sm.rowat[pos] = r;
        } else {
            g.flop[r] = 0;
            if (PRED) emit(r, 0);
        }
    }
    bar();

    // 3. segmented sum over the thread's entries: rows that start and end
    //    inside are written here; the head (before the first start) and the
    //    tail (from the last start) are combined across threads below
    const uint32_t bits = V == 32 ? sm.start[i0 >> 5] : (sm.start[i0 >> 5] >> (i0 & 31)) & ((1u << (V & 31)) - 1u);
    long long cur = 0, head = 0, tmax = 0;
    int32_t row = -1;
#pragma unroll
    for (int k = 0; k < V; ++k) {
        if ((bits >> k) & 1u) {
            if (row >= 0) {
                g.flop[row] = cur;  // complete inside the thread
                if (PRED) emit(row, cur);
                tmax = cur > tmax ? cur : tmax;
            } else {
                head = cur;
            }
            row = sm.rowat[i0 + k];
            cur = 0;
        }
        cur += d[k];
    }
    Carry mine;
    mine.flag = bits != 0u;
    mine.v = cur;  // tail value, or the whole thread when no row starts here
    mine.row = row;
    if (!mine.flag) head = cur;

    // 4. tile-wide exclusive segmented scan of the carries
    Carry inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const Carry u = shfl_up_carry(inc, o);
        if (lane >= o) inc = carry_op(u, inc);
    }
    if (lane == 31) sm.wc[warp] = inc;
    bar();
    Carry pre{0, 0, -1};  // carry entering this warp
    for (int w = 0; w < warp; ++w) pre = carry_op(pre, sm.wc[w]);
    Carry excl = shfl_up_carry(inc, 1);
    if (lane == 0) excl = Carry{0, 0, -1};
    const Carry cin = carry_op(pre, excl);  // carry entering this thread
    if (mine.flag) {
        // the carried row ends right before this thread's first start
        const long long v = cin.v + head;
        if (cin.flag) {
            g.flop[cin.row] = v;
            if (PRED) emit(cin.row, v);
            tmax = v > tmax ? v : tmax;
        } else {
            g.tile_lead[t] = v;  // continues a row owned by an earlier tile
        }
    }
    if (tid == BLOCK - 1) {
        const Carry all = carry_op(cin, mine);
        if (all.flag) {
            g.flop[all.row] = all.v;  // the fixup adds the following tiles' leading slices
            if (__ldg(&g.arpt[all.row + 1]) <= te) {  // the row ends with the tile: final
                tmax = all.v > tmax ? all.v : tmax;
                if (PRED) emit(all.row, all.v);
            }
        } else {
            g.tile_lead[t] = all.v;  // no row starts in this tile
        }
    }
    // (the scan's barrier orders the reuse of red / red2)
    (void)NW;
    tile_totals<BLOCK, V>(sm, g, t, tid, tsum, tmax, bar);
}

// One block per tile, degrees gathered from global memory (L2).
// (row mode holds a row's 16 gathers in flight: 64 registers, 8 blocks per SM)
template <int BLOCK, int V, bool PRED, bool ROWS, bool NOL1>
__global__ void __launch_bounds__(BLOCK, ROWS ? 8 : (SPNNZ_FLOP_MINB / BLOCK < 32 ? SPNNZ_FLOP_MINB / BLOCK : 32))
k_flop(TileArgs g, const uint16_t* __restrict__ bdeg, PredOut pred, int64_t t0) {
    __shared__ TileSmem<BLOCK, V> sm;
    Emit emit{};
    if (PRED) emit = make_emit(pred);
    if (g.prefetch_ahead && threadIdx.x == 0 && blockIdx.x + g.prefetch_ahead < gridDim.x)
        prefetch_tile(g, t0 + blockIdx.x + g.prefetch_ahead);
    flop_tile<BLOCK, V, PRED, ROWS>(sm, g, t0 + blockIdx.x, threadIdx.x, GlobalDeg<NOL1>{bdeg, policy_evict_last()},
                                    BlockBar{}, emit);
}

// Persistent blocks of G tile groups (G x 128 threads, one block per SM) with
// B's whole degree table in shared memory: loaded once per block, then every
// gather is a shared-memory load (config 4: K = 65536, 128 KB).  Each group
// runs the tile code on its own tiles with its own named barrier.
constexpr int kSmemGroups = 8;
template <int V, bool PRED, bool ROWS>
__global__ void __launch_bounds__(kFlopBlock * kSmemGroups, 1)
k_flop_smem(TileArgs g, const uint16_t* __restrict__ bdeg, int32_t k_rows, PredOut pred, int64_t t0,
            int64_t t1, unsigned long long* __restrict__ sched) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    auto* tiles = reinterpret_cast<TileSmem<kFlopBlock, V>*>(s_raw);
    uint16_t* s_deg = reinterpret_cast<uint16_t*>(s_raw + sizeof(TileSmem<kFlopBlock, V>) * kSmemGroups);
    const int grp = threadIdx.x / kFlopBlock, tid = threadIdx.x % kFlopBlock;
    // group g of block b takes tiles b G + g, + G gridDim, ... (static: a
    // same-address ticket counter serialises in L2); its next tile's columns
    // are L2-prefetched while it works on the current one
    const int64_t stride = int64_t(gridDim.x) * kSmemGroups;
    int64_t t = t0 + int64_t(blockIdx.x) * kSmemGroups + grp;
    if (tid == 0 && t < t1) prefetch_tile(g, t);
    // the degree table, 16 bytes per thread per step (k_rows padded to 8)
    const int words = (k_rows + 7) >> 3;
    for (int i = threadIdx.x; i < words; i += blockDim.x)
        reinterpret_cast<int4*>(s_deg)[i] = __ldg(reinterpret_cast<const int4*>(bdeg) + i);
    __syncthreads();
    Emit emit{};
    if (PRED) emit = make_emit(pred);
    const GroupBar<kFlopBlock> bar{1 + grp};
    for (; t < t1; t += stride) {
        if (tid == 0 && t + stride < t1) prefetch_tile(g, t + stride);
        flop_tile<kFlopBlock, V, PRED, ROWS>(tiles[grp], g, t, tid, SharedDeg{s_deg}, bar, emit);
    }
    (void)sched;
}

// ------------------------------------------------------------------
// Row blocks (A with short rows: config 4's A, a stencil): one warp per 32
// consecutive rows.  Their entries (contiguous in A.col) are copied into the
// warp's shared staging area with coalesced loads, then each lane sums ITS
// row from the staging -- so a warp's k-th gathers follow 32 consecutive rows
// (consecutive columns in a banded A) -- and writes it (32 consecutive int64
// per warp).  Rows end inside their block: no tile partition, no fixup; F and
// max go out with one pair of atomics per block.  A block whose entries
// exceed the staging area falls back to one row at a time (lane-strided).
// The degree table is in shared memory when B's rows fit (SMEM), else the
// L2-resident uint16 array.
constexpr int kRbRows = 32;
#ifndef SPNNZ_RB_STAGE
#define SPNNZ_RB_STAGE 1100
#endif
#ifndef SPNNZ_RB_MINB
#define SPNNZ_RB_MINB 3
#endif
#ifndef SPNNZ_RB_GV
#define SPNNZ_RB_GV 32
#endif
constexpr int kRbGv = SPNNZ_RB_GV;  // L2 degree gathers in flight per lane (row blocks)
template <bool SMEM>
struct RbShape {
    // SMEM: one 1024-thread block per SM beside the degree table; else
    // 256-thread blocks, several per SM
    static constexpr int kThreads = SMEM ? 1024 : 256;
    static constexpr int kWarps = kThreads / 32;
    // entries staged per warp: SMEM 32 x 640 x 4 B = 80 KB beside the table;
    // else 8 x 1100 x 4 B = 35.2 KB per block, three blocks (24 warps) per SM
    // whose lanes keep 32 degree gathers in flight (a stencil row's 27 in one
    // round; config 3: 82.7 -> 68 us, against 48 warps with 8 in flight)
    static constexpr int kStage = SMEM ? 640 : SPNNZ_RB_STAGE;
    static constexpr int kMinBlocks = SMEM ? 1 : SPNNZ_RB_MINB;
};

struct RbArgs {
    const int64_t* __restrict__ arpt;  // m + 1 absolute offsets
    const int32_t* __restrict__ acol;
    const int64_t* __restrict__ brpt;
    int32_t m;
    int64_t* __restrict__ flop;
    long long* __restrict__ totals;
    const unsigned* escapes;  // k_degree's flag: some B row has >= 65535 entries (nullable: assume so)
};

template <bool SMEM, bool PRED>
__global__ void __launch_bounds__(RbShape<SMEM>::kThreads, RbShape<SMEM>::kMinBlocks)
k_flop_rb(RbArgs g, const uint16_t* __restrict__ bdeg, int32_t k_rows, PredOut pred,
          unsigned long long* __restrict__ sched) {
    using Sh = RbShape<SMEM>;
    extern __shared__ __align__(16) unsigned char s_raw[];
    int32_t* stage_all = reinterpret_cast<int32_t*>(s_raw);
    const uint16_t* s_deg = reinterpret_cast<const uint16_t*>(s_raw + size_t(Sh::kWarps) * (Sh::kStage + 4) * 4);
    __shared__ long long s_sum[Sh::kWarps], s_max[Sh::kWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t* stage = stage_all + warp * (Sh::kStage + 4);  // (+ 4: the alignment shift)
    const uint64_t first = policy_evict_first(), last = policy_evict_last();
    if (SMEM) {
        uint16_t* d = const_cast<uint16_t*>(s_deg);
        const int words = (k_rows + 7) >> 3;
        for (int i = threadIdx.x; i < words; i += blockDim.x)
            reinterpret_cast<int4*>(d)[i] = __ldg(reinterpret_cast<const int4*>(bdeg) + i);
        __syncthreads();
    }
    Emit emit{};
    if (PRED) emit = make_emit(pred);
    const auto deg = [&](int32_t c) -> int32_t {
        SPNNZ_ASSERT(c >= 0 && c < k_rows);
        const int32_t v = SMEM ? s_deg[c] : gather_deg(bdeg + c, last);
        return v == 0xFFFF ? static_cast<int32_t>(__ldg(&g.brpt[c + 1]) - __ldg(&g.brpt[c])) : v;
    };
    const int64_t units = (int64_t(g.m) + kRbRows - 1) / kRbRows;
    const bool esc = g.escapes == nullptr || *g.escapes != 0u;  // uniform
    long long wsum = 0, wmax = 0;
    // SMEM: units handed out by a ticket counter (a block that starts late
    // takes fewer); else one unit per warp of the grid
    // every warp of the grid takes units warp, warp + W, ... (static: a
    // same-address ticket counter serialises in L2, ~one atomic per 15 ns)
    const int64_t ustride = int64_t(gridDim.x) * Sh::kWarps;
    int64_t u = int64_t(blockIdx.x) * Sh::kWarps + warp;
    // the row bounds of the warp's next unit are loaded one unit ahead
    int64_t rs_n = 0, re_n = 0;
    if (u < units && u * kRbRows + lane < g.m) {
        rs_n = __ldg(&g.arpt[u * kRbRows + lane]);
        re_n = __ldg(&g.arpt[u * kRbRows + lane + 1]);
    }
    for (; u < units; u += ustride) {
        const int32_t r0 = static_cast<int32_t>(u * kRbRows);
        const int32_t r = r0 + lane;
        const int32_t rl = r0 + kRbRows < g.m ? r0 + kRbRows : g.m;  // rows [r0, rl)
        const int64_t rs = rs_n, re = re_n;
        {
            const int64_t un = u + ustride, rn = un * kRbRows + lane;
            if (un < units && rn < g.m) {
                rs_n = __ldg(&g.arpt[rn]);
                re_n = __ldg(&g.arpt[rn + 1]);
            }
        }
        // rows [j, jend) whose entries fit the staging area go together; a
        // row longer than the area goes alone, lane-strided
        int32_t j = r0;
        while (j < rl) {
            const int64_t Ej = __shfl_sync(0xffffffffu, rs, j - r0);
            const unsigned fit = __ballot_sync(0xffffffffu, r >= j && r < rl && re - Ej <= Sh::kStage);
            if (fit == 0u) {  // row j alone
                const int64_t b = __shfl_sync(0xffffffffu, re, j - r0);
                long long sum = 0;
                for (int64_t e = Ej + lane; e < b; e += 32 * 4) {
                    int32_t c[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) c[k] = e + 32 * k < b ? ld_stream_i32(g.acol + e + 32 * k, first) : -1;
#pragma unroll
                    for (int k = 0; k < 4; ++k) sum += c[k] >= 0 ? deg(c[k]) : 0;
                }
                sum = warp_sum_ll(sum);
                if (lane == 0) {
                    g.flop[j] = sum;
                    if (PRED) emit(j, sum);
                    wsum += sum;
                    wmax = sum > wmax ? sum : wmax;
                }
                ++j;
                continue;
            }
            const int32_t jend = r0 + 32 - __clz(fit);  // rows [j, jend): a run of lanes
            const int64_t ne = __shfl_sync(0xffffffffu, re, jend - 1 - r0) - Ej;
            // stage their columns with asynchronous copies (every copy of the
            // run in flight at once, no registers), coalesced across the warp:
            // 16-byte L1-bypassing copies over the aligned body (entry e goes
            // to stage[sh + e - Ej], sh making the body's destinations 16-byte
            // aligned), 4-byte copies for the ragged head and tail
            int sh;
            {
                const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
                const int head0 = static_cast<int>(((16 - (reinterpret_cast<uintptr_t>(g.acol + Ej) & 15)) & 15) >> 2);
                const int h = head0 < ne ? head0 : static_cast<int>(ne);
                sh = (4 - h) & 3;
                const int nb = static_cast<int>((ne - h) >> 2);
                const int tail = static_cast<int>(ne - h - 4 * nb);
                if (lane < h + tail) {  // head and tail entries
                    const int e = lane < h ? lane : h + 4 * nb + (lane - h);
                    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(
                                     dst + 4u * static_cast<uint32_t>(sh + e)),
                                 "l"(g.acol + Ej + e), "l"(first)
                                 : "memory");
                }
                for (int cch = lane; cch < nb; cch += 32)
                    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(
                                     dst + 4u * static_cast<uint32_t>(sh + h + 4 * cch)),
                                 "l"(g.acol + Ej + h + 4 * cch), "l"(first)
                                 : "memory");
                asm volatile("cp.async.wait_all;" ::: "memory");
            }
            __syncwarp();
            if (r >= j && r < jend) {
                long long sum = 0;
                const int i0 = sh + static_cast<int>(rs - Ej), i1 = sh + static_cast<int>(re - Ej);
                if (!esc) {
                    // no escapes: a row of <= kStage entries sums in 32 bits
                    // (< 2^11 x 2^16) and every degree is the table's
                    int acc = 0;
                    if (SMEM) {
#pragma unroll 4
                        for (int i = i0; i < i1; ++i) acc += s_deg[stage[i]];
                    } else {
                        for (int i = i0; i < i1; i += kRbGv) {
                            int32_t d[kRbGv];
#pragma unroll
                            for (int k = 0; k < kRbGv; ++k)
                                d[k] = i + k < i1 ? static_cast<int32_t>(gather_deg(bdeg + stage[i + k], last)) : 0;
#pragma unroll
                            for (int k = 0; k < kRbGv; ++k) acc += d[k];
                        }
                    }
                    sum = acc;
                } else {
                    for (int i = i0; i < i1; i += 8) {
                        int32_t cc[8], d[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) cc[k] = i + k < i1 ? stage[i + k] : -1;
#pragma unroll
                        for (int k = 0; k < 8; ++k) d[k] = cc[k] >= 0 ? deg(cc[k]) : 0;
#pragma unroll
                        for (int k = 0; k < 8; ++k) sum += d[k];
                    }
                }
                g.flop[r] = sum;
                if (PRED) emit(r, sum);
                wsum += sum;
                wmax = sum > wmax ? sum : wmax;
            }
            __syncwarp();  // the staging is reused next
            j = jend;
        }
    }
    wsum = warp_sum_ll(wsum);
    wmax = warp_max_ll(wmax);
    if (lane == 0) {
        s_sum[warp] = wsum;
        s_max[warp] = wmax;
    }
    __syncthreads();
    if (warp == 0) {
        long long a = lane < Sh::kWarps ? s_sum[lane] : 0, b = lane < Sh::kWarps ? s_max[lane] : 0;
        a = warp_sum_ll(a);
        b = warp_max_ll(b);
        if (lane == 0) {
            if (a) atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[kF]), static_cast<unsigned long long>(a));
            atomicMax(reinterpret_cast<unsigned long long*>(&g.totals[kMax]), static_cast<unsigned long long>(b));
        }
    }
    (void)sched;
}

// ------------------------------------------------------------------
// Row streams (B's degree table in shared memory): each warp owns a
// contiguous range of rows [R0, R1) and streams their entries [E0, E1) as
// 128-entry chunks -- lane l loads entries c + 4l .. c + 4l + 3 with one
// aligned 16-byte load, kRsAhead chunks ahead of the one being summed, so
// A.col is read once, coalesced, with ~2 KB in flight per warp.  Per chunk:
// the four degrees (shared-memory gathers, masked outside [E0, E1)), and a
// warp inclusive scan of the lane sums, which gives P(x) = sum of the degrees
// over [E0, x) at every entry of the chunk.  The rows are taken 32 at a time
// (lane l owns row rb + l); an owner whose row ends inside the chunk reads
// P(end) from the lane holding the row's last entry (three shuffles: that
// lane's inclusive sum and its last three degrees packed), and a row's FLOP
// is P(end) - P(end of the previous row).  The shared pipe sees ~4 gathers
// and ~10 shuffles per 128 entries, where the staged row-per-lane walk
// (k_flop_rb) spent two bank-conflicted loads per entry and ran each warp
// as long as its longest row (config 4: 6.35 M shared wavefronts, 78 % of
// the L1 pipe).  ESC: some B row has >= 65535 entries -- degrees escape to
// B.rpt and the sums run in 64 bits (k_degree's flag picks the variant).
constexpr int kRsThreads = 1024;
#ifndef SPNNZ_RS_AHEAD
#define SPNNZ_RS_AHEAD 3
#endif
constexpr int kRsAhead = SPNNZ_RS_AHEAD;  // chunks in flight per warp (4: spills at 64 registers)
#ifndef SPNNZ_RS_AHEAD8
#define SPNNZ_RS_AHEAD8 2
#endif
constexpr int kRsAhead8 = SPNNZ_RS_AHEAD8;  // 256-entry chunks in flight per warp (fast path)
constexpr int kRsScratch = kRsThreads / 32 * 256 * 4;  // the fast path's per-warp query scratch (bytes)
struct RsArgs {
    const int64_t* __restrict__ arpt;  // m + 1 absolute offsets
    const int32_t* __restrict__ acol;  // indexed with absolute offsets
    const int64_t* __restrict__ brpt;
    int64_t lo, hi;  // absolute entry range backed by acol's allocation
    int32_t m;
    int32_t warps;  // warps sharing the rows (a contiguous range each)
    int64_t* __restrict__ flop;
    long long* __restrict__ totals;
    const unsigned* escapes;  // k_degree's flag (nullable: assume escapes)
    int32_t k_rows;           // B's rows (the degree table's length; bounds checks)
};

template <bool PRED, bool ESC>
__device__ __forceinline__ void rs_warp(const RsArgs& g, const uint16_t* s_deg, int32_t R0, int32_t R1,
                                        const Emit& emit, long long& wsum, long long& wmax) {
    using S = typename std::conditional<ESC, long long, int>::type;
    const int lane = threadIdx.x & 31;
    const uint64_t first = policy_evict_first();
    const int64_t E0 = __ldg(&g.arpt[R0]);
    // positions are 32-bit offsets from a0, the 16-byte aligned address at or
    // below E0 (chunk starts stay aligned; the launcher keeps A's entries
    // under 2^31 - 2^16)
    const int64_t a0 = E0 - static_cast<int64_t>((reinterpret_cast<uintptr_t>(g.acol + E0) & 15) >> 2);
    const int32_t* col0 = g.acol + a0;
    const int e0 = static_cast<int>(E0 - a0), e1 = static_cast<int>(__ldg(&g.arpt[R1]) - a0);
    const int lo = static_cast<int>(g.lo - a0 > -(1 << 30) ? g.lo - a0 : -(1 << 30));
    const int hi = static_cast<int>(g.hi - a0);
    // chunk loads: unguarded when the whole chunk lies inside the allocation
    const auto load = [&](int c) -> int4 {
        const int p = c + 4 * lane;
        if (c >= lo && c + 128 <= hi) return ld_stream_v4(reinterpret_cast<const int4*>(col0 + p), first);
        int4 v = make_int4(0, 0, 0, 0);
        if (c >= e1) return v;
        if (p >= lo && p < hi) v.x = ld_stream_i32(col0 + p, first);
        if (p + 1 >= lo && p + 1 < hi) v.y = ld_stream_i32(col0 + p + 1, first);
        if (p + 2 >= lo && p + 2 < hi) v.z = ld_stream_i32(col0 + p + 2, first);
        if (p + 3 >= lo && p + 3 < hi) v.w = ld_stream_i32(col0 + p + 3, first);
        return v;
    };
    const auto deg = [&](int32_t c) -> S {
        SPNNZ_ASSERT(c >= 0 && c < g.k_rows);
        const S v = s_deg[c];
        if (ESC && v == 0xFFFF) return static_cast<S>(__ldg(&g.brpt[c + 1]) - __ldg(&g.brpt[c]));
        return v;
    };
    // the current 32 rows [rb, rb + 32): lane's row end, resolved flag, P(end);
    // the next 32 rows' ends are loaded one group ahead (kept raw: converted
    // when used, so the load's latency stays hidden)
    int32_t rb = R0;
    bool valid = rb + lane < R1;
    int re = valid ? static_cast<int>(__ldg(&g.arpt[rb + lane + 1]) - a0) : e1;
    int64_t re_next = rb + 32 + lane < R1 ? __ldg(&g.arpt[rb + 32 + lane + 1]) : a0 + e1;
    bool res = !valid || re <= 0;  // (re <= 0 only for empty rows at E0 == a0: P = 0)
    long long pend = 0;
    long long carry = 0;  // P(end of the row before rb)
    long long base = 0;   // P(c)
    bool done = R0 >= R1;
    // the 32 rows are all resolved: write them, move to the next 32 (whose
    // rows ending at or before c -- empty rows at the stream's start -- have
    // P(end) = base)
    const auto advance = [&](int c) {
        long long prev = __shfl_up_sync(0xffffffffu, pend, 1);
        if (lane == 0) prev = carry;
        if (valid) {
            const long long sum = pend - prev;
            g.flop[rb + lane] = sum;
            if (PRED) emit(rb + lane, sum);
            wsum += sum;
            wmax = sum > wmax ? sum : wmax;
        }
        carry = __shfl_sync(0xffffffffu, pend, 31);
        rb += 32;
        done = rb >= R1;
        valid = rb + lane < R1;
        re = valid ? static_cast<int>(re_next - a0) : e1;
        re_next = rb + 32 + lane < R1 ? __ldg(&g.arpt[rb + 32 + lane + 1]) : a0 + e1;
        res = !valid || re <= c;
        pend = base;
    };
    int4 buf[kRsAhead];
#pragma unroll
    for (int k = 0; k < kRsAhead; ++k) buf[k] = load(128 * k);
    for (int c0 = 0; c0 < e1; c0 += 128 * kRsAhead) {
#pragma unroll
        for (int k = 0; k < kRsAhead; ++k) {
            const int c = c0 + 128 * k;
            const int4 v = buf[k];
            buf[k] = load(c + 128 * kRsAhead);
            if (c >= e1 || done) continue;  // warp-uniform
            S d0, d1, d2, d3;
            if (c >= e0 && c + 128 <= e1) {  // interior chunk (warp-uniform): no masking
                d0 = deg(v.x);
                d1 = deg(v.y);
                d2 = deg(v.z);
                d3 = deg(v.w);
            } else {
                const int p = c + 4 * lane;
                d0 = p >= e0 && p < e1 ? deg(v.x) : 0;
                d1 = p + 1 >= e0 && p + 1 < e1 ? deg(v.y) : 0;
                d2 = p + 2 >= e0 && p + 2 < e1 ? deg(v.z) : 0;
                d3 = p + 3 >= e0 && p + 3 < e1 ? deg(v.w) : 0;
            }
            S incl = d0 + d1 + d2 + d3;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const S t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const S total = __shfl_sync(0xffffffffu, incl, 31);
            for (;;) {
                // rows ending in (c, c + 128]: P(end) from the lane holding
                // the row's last entry (index q of the chunk)
                const bool q = !res && re <= c + 128;
                const int qi = q ? re - c - 1 : 4 * lane + 3;
                const int src = qi >> 2, j = qi & 3;
                S x;
                if (!ESC) {
                    const S top = __shfl_sync(0xffffffffu, incl, src);
                    const unsigned pk = __shfl_sync(0xffffffffu, static_cast<unsigned>(d3) |
                                                                     (static_cast<unsigned>(d2) << 16), src);
                    const S e1v = __shfl_sync(0xffffffffu, d1, src);
                    x = top - (j < 3 ? static_cast<S>(pk & 0xFFFFu) : 0) - (j < 2 ? static_cast<S>(pk >> 16) : 0) -
                        (j < 1 ? e1v : 0);
                } else {
                    const S top = __shfl_sync(0xffffffffu, incl, src);
                    const S e3 = __shfl_sync(0xffffffffu, d3, src);
                    const S e2 = __shfl_sync(0xffffffffu, d2, src);
                    const S e1v = __shfl_sync(0xffffffffu, d1, src);
                    x = top - (j < 3 ? e3 : 0) - (j < 2 ? e2 : 0) - (j < 1 ? e1v : 0);
                }
                if (q) {
                    pend = base + x;
                    res = true;
                }
                if (!__all_sync(0xffffffffu, res)) break;
                advance(c);
                if (done) break;
            }
            base += total;
        }
    }
    // no entries left: the remaining rows are empty and end at E1
    while (!done) {
        if (!res) pend = base;
        advance(e1);
    }
}

// The fast path (no escapes): 256-entry chunks, lane l holding entries
// c + 8l .. c + 8l + 7 from one 32-byte load, so the scan, the row queries
// and the loop cost half as much per entry.  Each lane publishes the prefix
// P(c + i + 1) - P(c) of its eight entries to the warp's 1 KB of shared
// scratch (two 16-byte stores, lane-contiguous: 4 wavefronts each) and an
// owner whose row ends at entry q of the chunk reads scratch slot q.  A.col
// buffers carry kColPad entries of tail padding, so a chunk is always loaded
// whole (entries outside [E0, E1) are masked before their gather).
constexpr int kRsChunk = 256;
__device__ __forceinline__ int rs_slot(int q) { return ((q & 4) << 5) + ((q >> 3) << 2) + (q & 3); }

template <bool PRED, class Bar>
__device__ __forceinline__ void rs_warp_fast(const RsArgs& g, const uint16_t* s_deg, int* xs, int32_t R0,
                                             int32_t R1, const Emit& emit, long long& wsum, long long& wmax,
                                             const Bar& table_ready) {
    const int lane = threadIdx.x & 31;
    const uint64_t first = policy_evict_first();
    const int64_t E0 = __ldg(&g.arpt[R0]);
    // 32-bit offsets from a0, the 32-byte aligned address at or below E0
    const int64_t a0 = E0 - static_cast<int64_t>((reinterpret_cast<uintptr_t>(g.acol + E0) & 31) >> 2);
    const int32_t* col0 = g.acol + a0 + 8 * lane;
    const int e0 = static_cast<int>(E0 - a0), e1 = static_cast<int>(__ldg(&g.arpt[R1]) - a0);
    struct V8 {
        int v[8];
    };
    const auto load = [&](int c) -> V8 {
        V8 r;
        if (c < e1) {
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                         : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
                           "=r"(r.v[6]), "=r"(r.v[7])
                         : "l"(col0 + c), "l"(first));
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) r.v[k] = 0;
        }
        return r;
    };
    // row ends, one group of 32 ahead: loaded unconditionally (index clamped
    // to R1, the value replaced at use) so no select waits on a load in
    // flight
    const auto end_at = [&](int32_t r) -> int64_t { return __ldg(&g.arpt[(r < R1 ? r : R1 - 1) + 1]); };
    int32_t rb = R0;
    bool valid = rb + lane < R1;
    const int64_t re_raw = end_at(rb + lane);
    int64_t re_next = end_at(rb + 32 + lane);
    V8 buf[kRsAhead8];
#pragma unroll
    for (int k = 0; k < kRsAhead8; ++k) buf[k] = load(kRsChunk * k);
    table_ready();  // the block's degree table has landed (the loads above overlap its copy)
    int re = valid ? static_cast<int>(re_raw - a0) : e1;
    bool res = !valid || re <= 0;
    long long pend = 0, carry = 0, base = 0;
    bool done = R0 >= R1;
    const auto advance = [&](int c) {
        long long prev = __shfl_up_sync(0xffffffffu, pend, 1);
        if (lane == 0) prev = carry;
        if (valid) {
            const long long sum = pend - prev;
            g.flop[rb + lane] = sum;
            if (PRED) emit(rb + lane, sum);
            wsum += sum;
            wmax = sum > wmax ? sum : wmax;
        }
        carry = __shfl_sync(0xffffffffu, pend, 31);
        rb += 32;
        done = rb >= R1;
        valid = rb + lane < R1;
        re = valid ? static_cast<int>(re_next - a0) : e1;
        re_next = end_at(rb + 32 + lane);
        res = !valid || re <= c;
        pend = base;
    };
    for (int c0 = 0; c0 < e1; c0 += kRsChunk * kRsAhead8) {
#pragma unroll
        for (int k = 0; k < kRsAhead8; ++k) {
            const int c = c0 + kRsChunk * k;
            const V8 v = buf[k];
            buf[k] = load(c + kRsChunk * kRsAhead8);
            if (c >= e1 || done) continue;  // warp-uniform
            int x[8];
            if (c >= e0 && c + kRsChunk <= e1) {  // interior chunk: no masking
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    SPNNZ_ASSERT(v.v[i] >= 0 && v.v[i] < g.k_rows);
                    x[i] = s_deg[v.v[i]];
                }
            } else {
                const int p = c + 8 * lane;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const bool in = p + i >= e0 && p + i < e1;
                    SPNNZ_ASSERT(!in || (v.v[i] >= 0 && v.v[i] < g.k_rows));
                    x[i] = in ? s_deg[v.v[i]] : 0;
                }
            }
#pragma unroll
            for (int i = 1; i < 8; ++i) x[i] += x[i - 1];
            int incl = x[7];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            const int excl = incl - x[7];
            reinterpret_cast<int4*>(xs)[lane] = make_int4(excl + x[0], excl + x[1], excl + x[2], excl + x[3]);
            reinterpret_cast<int4*>(xs)[32 + lane] = make_int4(excl + x[4], excl + x[5], excl + x[6], excl + x[7]);
            __syncwarp();
            for (;;) {
                // rows ending in (c, c + 256]: P(end) = base + prefix through
                // the row's last entry
                if (!res && re <= c + kRsChunk) {
                    SPNNZ_ASSERT(re - c - 1 >= 0 && re - c - 1 < kRsChunk);
                    pend = base + xs[rs_slot(re - c - 1)];
                    res = true;
                }
                if (!__all_sync(0xffffffffu, res)) break;
                advance(c);
                if (done) break;
            }
            __syncwarp();  // the scratch is rewritten by the next chunk
            base += total;
        }
    }
    while (!done) {
        if (!res) pend = base;
        advance(e1);
    }
}

// the escape variant (64-bit sums, B rows of >= 65535 entries: rare)
template <bool PRED>
__device__ __forceinline__ void rs_warp_esc(const RsArgs& g, const uint16_t* s_deg, int32_t R0, int32_t R1,
                                         const Emit& emit, long long& wsum, long long& wmax) {
    rs_warp<PRED, true>(g, s_deg, R0, R1, emit, wsum, wmax);
}

template <bool PRED>
__global__ void __launch_bounds__(kRsThreads, 1)
k_flop_rs(RsArgs g, const uint16_t* __restrict__ bdeg, int32_t k_rows, PredOut pred) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    __shared__ long long s_sum[kRsThreads / 32], s_max[kRsThreads / 32];
    int* s_xs = reinterpret_cast<int*>(s_raw);  // kRsScratch bytes, then the table
    uint16_t* s_deg = reinterpret_cast<uint16_t*>(s_raw + kRsScratch);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    {
        // the degree table: asynchronous 16-byte copies, waited for after
        // each warp has queued its first loads
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(s_deg));
        const int words = (k_rows + 7) >> 3;
        for (int i = threadIdx.x; i < words; i += blockDim.x)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * i),
                         "l"(reinterpret_cast<const int4*>(bdeg) + i)
                         : "memory");
    }
    const auto table_ready = [] {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    };
    Emit emit{};
    if (PRED) emit = make_emit(pred);
    long long wsum = 0, wmax = 0;
    const int w = blockIdx.x * (kRsThreads / 32) + warp;
    const int32_t R0 = static_cast<int32_t>(int64_t(g.m) * w / g.warps);
    const int32_t R1 = static_cast<int32_t>(int64_t(g.m) * (w + 1) / g.warps);
    const bool esc = g.escapes == nullptr || *g.escapes != 0u;  // uniform
    if (w < g.warps && !esc) {
        rs_warp_fast<PRED>(g, s_deg, s_xs + warp * 256, R0, R1, emit, wsum, wmax, table_ready);
    } else {
        table_ready();
        if (w < g.warps) rs_warp_esc<PRED>(g, s_deg, R0, R1, emit, wsum, wmax);
    }
    wsum = warp_sum_ll(wsum);
    wmax = warp_max_ll(wmax);
    if (lane == 0) {
        s_sum[warp] = wsum;
        s_max[warp] = wmax;
    }
    __syncthreads();
    if (warp == 0) {
        long long a = s_sum[lane], b = s_max[lane];
        a = warp_sum_ll(a);
        b = warp_max_ll(b);
        if (lane == 0) {
            if (a) atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[kF]), static_cast<unsigned long long>(a));
            atomicMax(reinterpret_cast<unsigned long long*>(&g.totals[kMax]), static_cast<unsigned long long>(b));
        }
    }
}

// Adds each tile's leading slice to the row it continues (one thread per
// first continuing tile of a row, summing the run of tiles that continue the
// same row) and reduces F and max over all tiles.
template <int BLOCK, bool PRED>
__global__ void __launch_bounds__(BLOCK)
k_flop_fixup(const int32_t* __restrict__ tile_row, int64_t tiles,
             const long long* __restrict__ tile_lead, const long long* __restrict__ tile_total,
             const long long* __restrict__ tile_max, int64_t* __restrict__ flop,
             long long* __restrict__ totals, PredOut pred) {
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
            if (PRED) make_emit(pred)(r, v);
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

// FLOP of listed rows (compute_flop's sum, flop.hpp:41-50, for those rows),
// as a flat decomposition so no warp walks a long row step after dependent
// step: every row is cut into kItemChunk-entry chunks, a one-block scan
// numbers them, and one warp per chunk adds its sum into the row's slot.
// (Warps over rows of up to 2048 entries plus one block per hub row left the
// multi-GPU sampled-FLOP step at ~40 us, latency-bound.)
constexpr int kItemChunk = 128;  // one step of four loads per lane

// units[s] = chunks of item s (0 outside the shard); out[s] = 0
__global__ void __launch_bounds__(256) k_item_chunks(DevCsr a, int32_t row_lo, const int32_t* __restrict__ rows,
                                                    int64_t n, int64_t* __restrict__ units,
                                                    int64_t* __restrict__ out) {
    for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < n; s += int64_t(gridDim.x) * blockDim.x) {
        const int32_t r = rows[s] - row_lo;
        int64_t u = 0;
        if (r >= 0 && r < a.rows) u = (a.rpt[r + 1] - a.rpt[r] + kItemChunk - 1) / kItemChunk;
        units[s] = u;
        out[s] = 0;
    }
}

// In-place exclusive scan of units[0..n) by one block; units[n] = total.
// Thread t owns the contiguous run [t c, (t + 1) c), c = ceil(n / BLOCK),
// staged through shared memory when the list fits (coalesced loads and
// stores, one block scan of the run sums); a scan per BLOCK items made this a
// chain of barriers (~2 us per 1024 items).
constexpr int kScanSmemItems = 24576;  // 192 KB of int64

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_item_scan(int64_t* __restrict__ units, int64_t n) {
    using Scan = cub::BlockScan<long long, BLOCK>;
    __shared__ typename Scan::TempStorage tmp;
    extern __shared__ long long s_items[];
    const bool staged = n <= kScanSmemItems;
    long long* v = staged ? s_items : reinterpret_cast<long long*>(units);
    if (staged) {
        for (int64_t i = threadIdx.x; i < n; i += BLOCK) s_items[i] = units[i];
        __syncthreads();
    }
    const int64_t c = (n + BLOCK - 1) / BLOCK;
    const int64_t i0 = threadIdx.x * c, i1 = i0 + c < n ? i0 + c : n;
    long long sum = 0;
    for (int64_t i = i0; i < i1; ++i) sum += v[i];
    long long ex, tot;
    Scan(tmp).ExclusiveSum(sum, ex, tot);
    for (int64_t i = i0; i < i1; ++i) {
        const long long x = v[i];
        v[i] = ex;
        ex += x;
    }
    if (staged) {
        __syncthreads();
        for (int64_t i = threadIdx.x; i < n; i += BLOCK) units[i] = s_items[i];
    }
    if (threadIdx.x == 0) units[n] = tot;
}

__global__ void __launch_bounds__(256) k_item_flop(DevCsr a, const int64_t* __restrict__ brpt,
                                                  int32_t row_lo, const int32_t* __restrict__ rows,
                                                  int64_t n, const int64_t* __restrict__ pre,
                                                  int64_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long total = pre[n];
    for (long long u = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; u < total;
         u += (int64_t(gridDim.x) * blockDim.x) >> 5) {
        int64_t lo = 0, hi = n - 1;  // largest item with pre[item] <= u
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (__ldg(&pre[mid]) <= u) lo = mid; else hi = mid - 1;
        }
        const int32_t r = rows[lo] - row_lo;
        const int64_t e1 = a.rpt[r + 1];
        const int64_t c0 = a.rpt[r] + (u - pre[lo]) * kItemChunk;
        const int64_t c1 = c0 + kItemChunk < e1 ? c0 + kItemChunk : e1;
        long long f = 0;
        int c[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] = c0 + lane + 32 * k < c1 ? __ldg(&a.col[c0 + lane + 32 * k]) : -1;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (c[k] >= 0) f += __ldg(&brpt[c[k] + 1]) - __ldg(&brpt[c[k]]);
        f = warp_sum_ll(f);
        if (lane == 0 && f)
            atomicAdd(reinterpret_cast<unsigned long long*>(&out[lo]), static_cast<unsigned long long>(f));
    }
}

// Rank r counts the items whose FLOP prefix P[i] lies in [T_r, T_{r+1}),
// T_r = floor(total r / world) (the last rank also takes P[i] = total), so
// the ranks split the list into contiguous, FLOP-balanced windows whatever
// the order of heavy and light rows.  One block: the list is the sample.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_flop_window(const int64_t* __restrict__ f, int64_t n, int rank,
                                                      int world, int64_t* __restrict__ window) {
    using Scan = cub::BlockScan<long long, BLOCK>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ long long s_red[BLOCK / 32];
    extern __shared__ long long s_items[];
    const bool staged = n <= kScanSmemItems;  // coalesced loads, as k_item_scan
    const long long* v = staged ? s_items : reinterpret_cast<const long long*>(f);
    if (staged) {
        for (int64_t i = threadIdx.x; i < n; i += BLOCK) s_items[i] = f[i];
        __syncthreads();
    }
    const int64_t c = (n + BLOCK - 1) / BLOCK;  // thread t owns items [t c, (t + 1) c)
    const int64_t i0 = threadIdx.x * c, i1 = i0 + c < n ? i0 + c : n;
    long long sum = 0;
    for (int64_t i = i0; i < i1; ++i) sum += v[i];
    long long ex, total;
    Scan(tmp).ExclusiveSum(sum, ex, total);  // total is broadcast to every thread
    const auto split = [&](int r) -> long long {  // floor(total r / world) without overflow
        return (total / world) * r + (total % world) * r / world;
    };
    const long long t_lo = split(rank), t_hi = split(rank + 1);
    long long below_lo = 0, below_hi = 0;  // items with P[i] < T_r, < T_{r+1}
    for (int64_t i = i0; i < i1; ++i) {
        below_lo += ex < t_lo;
        below_hi += ex < t_hi;
        ex += v[i];
    }
    below_lo = block_sum_ll<BLOCK>(below_lo, s_red);  // valid in warp 0
    below_hi = block_sum_ll<BLOCK>(below_hi, s_red);
    if (threadIdx.x == 0) {
        window[0] = rank == 0 ? 0 : below_lo;
        window[1] = rank == world - 1 ? n : below_hi;
    }
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

// Banded-A check for the FLOP pass's row mode (sampled pairs of
// consecutive rows): out[0] pairs with both rows non-empty, out[1] of them
// whose first columns advance by 0..2 (a stencil's rows do), out[2] of them
// whose first row has <= 64 entries.
__global__ void k_locality(const int64_t* __restrict__ rpt, const int32_t* __restrict__ col, int32_t lo,
                           int32_t hi, int n, int* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || hi - lo < 2) return;
    const int32_t r = lo + static_cast<int32_t>((int64_t(hi - lo - 1) * i) / n);
    const int64_t a = rpt[r], b = rpt[r + 1], c = rpt[r + 2];
    if (b > a && c > b) {
        atomicAdd(&out[0], 1);
        const int d = col[b] - col[a];
        if (d >= 0 && d <= 2) atomicAdd(&out[1], 1);
        if (b - a <= 64) atomicAdd(&out[2], 1);
    }
}

// Instrumentation: the FLOP pass's loads with none of its row logic (the
// floor its access pattern sets on this matrix): 16 consecutive A.col entries
// per thread (the k_flop loads) and, with GATHER, their 16 degree gathers;
// one int64 written per thread so nothing is dead code.
template <bool GATHER, bool NOL1>
__global__ void __launch_bounds__(128, 10) k_pattern(const int32_t* __restrict__ col, int64_t base, int64_t nnz,
                                                   const uint16_t* __restrict__ deg, long long* __restrict__ out) {
    const uint64_t first = policy_evict_first(), last = policy_evict_last();
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int64_t e0 = ((base + 7) & ~int64_t(7)) + t * 16;
    if (e0 + 16 > base + nnz) return;
    int32_t c[16];
    // the tile kernel's loads: two 32-byte L1-bypassing loads per thread
#pragma unroll
    for (int k = 0; k < 2; ++k)
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                     : "=r"(c[8 * k]), "=r"(c[8 * k + 1]), "=r"(c[8 * k + 2]), "=r"(c[8 * k + 3]),
                       "=r"(c[8 * k + 4]), "=r"(c[8 * k + 5]), "=r"(c[8 * k + 6]), "=r"(c[8 * k + 7])
                     : "l"(col + e0 + 8 * k), "l"(first));
    long long s = 0;
    if (GATHER) {
        const GlobalDeg<NOL1> dg{deg, last};
        int32_t d[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) d[k] = dg(c[k]);
#pragma unroll
        for (int k = 0; k < 16; ++k) s += d[k];
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) s += c[k];
    }
    out[t] = s;
}

// The same instrumentation for the row-stream pass (k_flop_rs): one
// 1024-thread block per SM copies the uint16 degree table into shared memory,
// each warp streams a contiguous slice of A.col as 256-entry chunks (one
// 32-byte load per lane, kRsAhead8 chunks in flight) and, with GATHER, gathers
// the eight degrees of each from the shared table.  No row logic (no scan, no
// scratch, no A.rpt, no flop written): the floor the loads and the shared
// gathers set for that kernel's shape.
template <bool GATHER>
__global__ void __launch_bounds__(kRsThreads, 1)
k_pattern_table(const int32_t* __restrict__ col, int64_t base, int64_t nnz, const uint16_t* __restrict__ bdeg,
                int32_t k_rows, long long* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    uint16_t* s_deg = reinterpret_cast<uint16_t*>(s_raw + kRsScratch);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (GATHER) {
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(s_deg));
        const int words = (k_rows + 7) >> 3;
        for (int i = threadIdx.x; i < words; i += blockDim.x)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * i),
                         "l"(reinterpret_cast<const int4*>(bdeg) + i)
                         : "memory");
    }
    const uint64_t first = policy_evict_first();
    const int64_t warps = int64_t(gridDim.x) * (kRsThreads / 32);
    const int64_t w = blockIdx.x * int64_t(kRsThreads / 32) + warp;
    // whole 256-entry chunks, 32-byte aligned, split evenly over the warps
    const int64_t a0 = (base + 7) & ~int64_t(7);
    const int64_t chunks = (base + nnz - a0) / kRsChunk;
    const int64_t c_lo = chunks * w / warps, c_hi = chunks * (w + 1) / warps;
    const int32_t* p = col + a0 + c_lo * kRsChunk + 8 * lane;
    const int n = static_cast<int>(c_hi - c_lo);
    struct V8 {
        int v[8];
    };
    const auto load = [&](int c) -> V8 {
        V8 r;
        if (c < n) {
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                         : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
                           "=r"(r.v[6]), "=r"(r.v[7])
                         : "l"(p + int64_t(c) * kRsChunk), "l"(first));
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) r.v[k] = 0;
        }
        return r;
    };
    V8 buf[kRsAhead8];
#pragma unroll
    for (int k = 0; k < kRsAhead8; ++k) buf[k] = load(k);
    if (GATHER) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    }
    long long s = 0;
    for (int c0 = 0; c0 < n; c0 += kRsAhead8) {
#pragma unroll
        for (int k = 0; k < kRsAhead8; ++k) {
            const V8 v = buf[k];
            buf[k] = load(c0 + k + kRsAhead8);
            if (c0 + k >= n) continue;
            int x = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) x += GATHER ? static_cast<int>(s_deg[v.v[i]]) : v.v[i];
            s += x;
        }
    }
    out[blockIdx.x * int64_t(kRsThreads) + threadIdx.x] = s;
}

}  // namespace

cudaError_t launch_pattern(const DevCsr& a, const uint16_t* deg, bool gather, bool nol1, long long* out,
                           cudaStream_t stream) {
    const int64_t threads = a.nnz / 16;
    if (threads < 1) return cudaSuccess;
    const unsigned grid = static_cast<unsigned>((threads + 127) / 128);
    if (gather && nol1)
        k_pattern<true, true><<<grid, 128, 0, stream>>>(a.col, a.base, a.nnz, deg, out);
    else if (gather)
        k_pattern<true, false><<<grid, 128, 0, stream>>>(a.col, a.base, a.nnz, deg, out);
    else
        k_pattern<false, false><<<grid, 128, 0, stream>>>(a.col, a.base, a.nnz, deg, out);
    return cudaGetLastError();
}

cudaError_t launch_locality(const int64_t* rpt, const int32_t* col, int32_t lo, int32_t hi, int n, int* out3,
                            cudaStream_t stream) {
    cudaMemsetAsync(out3, 0, 3 * sizeof(int), stream);
    k_locality<<<(n + 255) / 256, 256, 0, stream>>>(rpt, col, lo, hi, n, out3);
    return cudaGetLastError();
}

cudaError_t launch_flop_window(const int64_t* item_flop, int64_t n, int rank, int world, int64_t* window,
                               cudaStream_t stream) {
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_done.load(std::memory_order_acquire) & (1ull << (dev & 63)))) {
        cudaFuncSetAttribute(k_flop_window<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, kScanSmemItems * 8);
        cudaFuncSetAttribute(k_item_scan<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, kScanSmemItems * 8);
        attr_done.fetch_or(1ull << (dev & 63), std::memory_order_release);
    }
    const size_t smem = n <= kScanSmemItems ? size_t(n) * 8 : 0;
    k_flop_window<1024><<<1, 1024, smem, stream>>>(item_flop, n, rank, world, window);
    return cudaGetLastError();
}

cudaError_t launch_item_flop(const DevCsr& a, const int64_t* brpt, int32_t row_lo,
                             const int32_t* rows, int64_t n, int64_t* out, int64_t* units, int num_sms,
                             cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    int64_t g1 = (n + 255) / 256;
    if (g1 > int64_t(num_sms) * 4) g1 = int64_t(num_sms) * 4;
    k_item_chunks<<<static_cast<unsigned>(g1), 256, 0, stream>>>(a, row_lo, rows, n, units, out);
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_done.load(std::memory_order_acquire) & (1ull << (dev & 63)))) {
        cudaFuncSetAttribute(k_item_scan<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, kScanSmemItems * 8);
        attr_done.fetch_or(1ull << (dev & 63), std::memory_order_release);
    }
    k_item_scan<1024><<<1, 1024, n <= kScanSmemItems ? size_t(n) * 8 : 0, stream>>>(units, n);
    k_item_flop<<<static_cast<unsigned>(num_sms) * 8, 256, 0, stream>>>(a, brpt, row_lo, rows, n, units, out);
    return cudaGetLastError();
}

__global__ void k_predict_redo(const int64_t* __restrict__ flop, int64_t m, PredOut p) {
    const double cr = predicted_cr(p.totals[kFStar], p.totals[kZStar]);
    const unsigned long long n = *p.nredo;
    const bool all = n > static_cast<unsigned long long>(p.redo_cap);
    const int64_t cnt = all ? m : static_cast<int64_t>(n);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < cnt;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = all ? i : p.redo[i];
        double q;
        const long long c = ceil_view(flop[r], cr, &q);
        if (p.ceil) p.ceil[r] = c;
        if (p.real) p.real[r] = q;
    }
}

cudaError_t launch_predict_redo(const int64_t* flop, int64_t m, const PredOut& pred, int num_sms,
                                cudaStream_t stream) {
    if (!pred.on() || m == 0) return cudaSuccess;
    k_predict_redo<<<static_cast<unsigned>(num_sms) * 4, 256, 0, stream>>>(flop, m, pred);
    return cudaGetLastError();
}

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

static TileMarks tile_marks(const DevCsr& a, const FlopScratch& s, int64_t a_off) {
    TileMarks mk;
    mk.tile_row = s.tile_x;
    mk.a_off = a_off;
    mk.m = a.rows;
    mk.base = a.base;
    mk.tiles = flop_tiles(a);
    return mk;
}

static unsigned stream_grid(int64_t n, int num_sms) {
    int64_t grid = (n + 255) / 256;
    if (grid > int64_t(num_sms) * 16) grid = int64_t(num_sms) * 16;
    return static_cast<unsigned>(grid < 1 ? 1 : grid);
}

cudaError_t launch_degree(const int64_t* brpt, int64_t k_rows, uint16_t* deg, int num_sms,
                          cudaStream_t stream, const DevCsr* a, const FlopScratch* s, int64_t* launches,
                          unsigned* escapes) {
    // A's partition rides along when A.rpt is a view into B.rpt
    const bool fuse = a && s && a->rows > 0 && a->rpt >= brpt && a->rpt + a->rows <= brpt + k_rows;
    if (k_rows == 0 && !(a && s)) return cudaSuccess;
    if (a && s && a->rows > 0 && !fuse) {
        k_tile_rows<<<stream_grid(a->rows, num_sms), 256, 0, stream>>>(a->rpt, tile_marks(*a, *s, 0));
        if (launches) ++*launches;
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (k_rows == 0) return cudaSuccess;
    const TileMarks mk = fuse ? tile_marks(*a, *s, a->rpt - brpt) : TileMarks();
    if (reinterpret_cast<uintptr_t>(brpt) & 15) return cudaErrorMisalignedAddress;  // cudaMalloc'd
    // (escapes: zeroed by the caller once per loaded B -- the flag only ever
    // goes 0 -> 1 for the same B, so no per-call reset is needed)
    k_degree<<<stream_grid((k_rows + 3) / 4, num_sms), 256, 0, stream>>>(brpt, k_rows, deg, mk, escapes);
    if (launches) ++*launches;
    return cudaGetLastError();
}

#ifdef SPNNZ_BINARY_PARTITION
cudaError_t launch_flop_partition(const DevCsr& a, const FlopScratch& s, cudaStream_t stream) {
    const int64_t tiles = flop_tiles(a);
    if (tiles == 0) return cudaSuccess;
    const int block = 256;
    const int64_t grid = (tiles + 1 + block - 1) / block;
    k_flop_partition<<<static_cast<unsigned>(grid), block, 0, stream>>>(a.rpt, a.rows, a.base,
                                                                      a.nnz, tiles, s.tile_x);
    return cudaGetLastError();
}
#endif

// the FLOP kernel the calling thread launched last (instrumentation)
static thread_local const char* g_last_kernel = "";
const char* last_flop_kernel() { return g_last_kernel; }

// dynamic shared memory of k_flop_smem; its static part (the ticket slots)
// is kept under kSmemStatic, and the total under the 227 KB per-block limit
constexpr size_t kSmemStatic = 1024;
static size_t flop_smem_bytes(int32_t k_rows) {
    return sizeof(TileSmem<kFlopBlock, kFlopIpt>) * kSmemGroups + ((size_t(k_rows) * 2 + 15) & ~size_t(15));
}

// K <= 81280 rows (tests/test_gpu_parity.py and bench.py name this limit)
bool flop_smem_fits(int32_t k_rows) {
    return k_rows > 0 && flop_smem_bytes(k_rows) + kSmemStatic <= 227 * 1024;
}

static TileArgs tile_args(const DevCsr& a, const int64_t* brpt, const FlopScratch& s, int64_t* flop,
                          const FlopMode& mode) {
    TileArgs g;
    g.arpt = a.rpt;
    g.acol = a.col;
    g.brpt = brpt;
    g.base = a.base;
    g.nnz = a.nnz;
    g.tile_row = s.tile_x;
    g.flop = flop;
    g.tile_lead = s.tile_carry;
    g.tile_total = s.tile_total;
    g.tile_max = s.tile_max;
    g.prefetch_ahead = mode.prefetch_ahead;
    return g;
}

template <bool PRED, bool ROWS, bool NOL1 = false>
static cudaError_t launch_tiles(const TileArgs& g, const uint16_t* bdeg, int64_t t_begin, int64_t t_end,
                                cudaStream_t stream, const PredOut& pred, const FlopMode& mode) {
    if (flop_smem_fits(mode.b_rows) && !mode.no_smem) {
        const size_t smem = flop_smem_bytes(mode.b_rows);
        static std::atomic<unsigned long long> attr_done{0};
        int dev = 0;
        cudaGetDevice(&dev);
        if (!(attr_done.load(std::memory_order_acquire) & (1ull << (dev & 63)))) {
            cudaFuncSetAttribute(k_flop_smem<kFlopIpt, PRED, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(227 * 1024 - kSmemStatic));
            attr_done.fetch_or(1ull << (dev & 63), std::memory_order_release);
        }
        int64_t grid = (t_end - t_begin + kSmemGroups - 1) / kSmemGroups;
        if (grid > mode.num_sms) grid = mode.num_sms;
        g_last_kernel = "k_flop_smem (tile groups, degree table in shared memory)";
        k_flop_smem<kFlopIpt, PRED, ROWS><<<static_cast<unsigned>(grid), kFlopBlock * kSmemGroups, smem, stream>>>(
            g, bdeg, mode.b_rows, pred, t_begin, t_end, mode.sched);
    } else {
        g_last_kernel = ROWS ? "k_flop (row-mode tiles, degree gathers from L2)" : "k_flop (tiles, degree gathers from L2)";
        // A/B knob: the shared-memory carve-out (percent of the SM's 228 KB;
        // the rest is L1 for the degree gathers): fewer resident tile blocks,
        // more L1.  Unset: the driver sizes it for the most resident blocks.
        static const int carve = [] {
            const char* e = getenv("SPNNZ_FLOP_CARVEOUT");
            return e ? atoi(e) : -1;
        }();
        if (carve >= 0) {
            static std::atomic<unsigned long long> carve_done{0};
            int dev = 0;
            cudaGetDevice(&dev);
            if (!(carve_done.load(std::memory_order_acquire) & (1ull << (dev & 63)))) {
                cudaFuncSetAttribute(k_flop<kFlopBlock, kFlopIpt, PRED, ROWS, NOL1>,
                                     cudaFuncAttributePreferredSharedMemoryCarveout, carve);
                carve_done.fetch_or(1ull << (dev & 63), std::memory_order_release);
            }
        }
        k_flop<kFlopBlock, kFlopIpt, PRED, ROWS, NOL1><<<static_cast<unsigned>(t_end - t_begin), kFlopBlock, 0, stream>>>(
            g, bdeg, pred, t_begin);
    }
    return cudaGetLastError();
}

cudaError_t launch_flop_tiles(const DevCsr& a, const uint16_t* bdeg, const int64_t* brpt,
                              const FlopScratch& s, int64_t* flop, int64_t t_begin, int64_t t_end,
                              cudaStream_t stream, const PredOut& pred, const FlopMode& mode) {
    if (t_end <= t_begin) return cudaSuccess;
    const TileArgs g = tile_args(a, brpt, s, flop, mode);
    if (mode.rows_mode)
        return pred.on() ? launch_tiles<true, true>(g, bdeg, t_begin, t_end, stream, pred, mode)
                         : launch_tiles<false, true>(g, bdeg, t_begin, t_end, stream, pred, mode);
    if (mode.gather_nol1)
        return pred.on() ? launch_tiles<true, false, true>(g, bdeg, t_begin, t_end, stream, pred, mode)
                         : launch_tiles<false, false, true>(g, bdeg, t_begin, t_end, stream, pred, mode);
    return pred.on() ? launch_tiles<true, false>(g, bdeg, t_begin, t_end, stream, pred, mode)
                     : launch_tiles<false, false>(g, bdeg, t_begin, t_end, stream, pred, mode);
}

template <bool SMEM, bool PRED>
static cudaError_t launch_rb(const RbArgs& g, const uint16_t* bdeg, int32_t k_rows, const PredOut& pred,
                             const FlopMode& mode, cudaStream_t stream) {
    using Sh = RbShape<SMEM>;
    const size_t smem = size_t(Sh::kWarps) * (Sh::kStage + 4) * 4 + (SMEM ? ((size_t(k_rows) * 2 + 15) & ~size_t(15)) : 0);
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_done.load(std::memory_order_acquire) & (1ull << (dev & 63)))) {
        cudaFuncSetAttribute(k_flop_rb<SMEM, PRED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(227 * 1024 - kSmemStatic));
        attr_done.fetch_or(1ull << (dev & 63), std::memory_order_release);
    }
    const int64_t units = (int64_t(g.m) + kRbRows - 1) / kRbRows;
    // persistent: one wave of blocks, every warp striding over the units (the
    // next unit's row bounds are loaded while the current one is summed)
    int64_t grid = (units + Sh::kWarps - 1) / Sh::kWarps;
    const int64_t wave = int64_t(mode.num_sms) * Sh::kMinBlocks;
    if (grid > wave && (SMEM || mode.rb_persistent)) grid = wave;
    if (grid < 1) grid = 1;
    g_last_kernel = SMEM ? "k_flop_rb (staged row blocks, degree table in shared memory)"
                         : "k_flop_rb (row blocks, degree gathers from L2)";
    k_flop_rb<SMEM, PRED><<<static_cast<unsigned>(grid), Sh::kThreads, smem, stream>>>(g, bdeg, k_rows, pred,
                                                                                       mode.sched);
    return cudaGetLastError();
}

// the staged row-block kernel's table limit (K <= 74496: the A/B reference)
static bool flop_rb_staged_fits(int32_t k_rows) {
    using Sh = RbShape<true>;
    return k_rows > 0 && size_t(Sh::kWarps) * (Sh::kStage + 4) * 4 + ((size_t(k_rows) * 2 + 15) & ~size_t(15)) +
                             kSmemStatic <= 227 * 1024;
}

static size_t flop_rs_smem_bytes(int32_t k_rows) { return kRsScratch + ((size_t(k_rows) * 2 + 15) & ~size_t(15)); }

// row streams: the query scratch and the table (K <= 99328)
bool flop_rb_smem_fits(int32_t k_rows) {
    return k_rows > 0 && flop_rs_smem_bytes(k_rows) + kSmemStatic <= 227 * 1024;
}

static bool flop_rs_on() {
    const char* e = getenv("SPNNZ_FLOP_RS");  // A/B knob: 0 = the staged row blocks
    return !(e && atoi(e) == 0);
}

template <bool PRED>
static cudaError_t launch_rs(const RsArgs& g0, const uint16_t* bdeg, int32_t k_rows, const PredOut& pred,
                             const FlopMode& mode, cudaStream_t stream) {
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_done.load(std::memory_order_acquire) & (1ull << (dev & 63)))) {
        cudaFuncSetAttribute(k_flop_rs<PRED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(227 * 1024 - kSmemStatic));
        attr_done.fetch_or(1ull << (dev & 63), std::memory_order_release);
    }
    RsArgs g = g0;
    // one 1024-thread block per SM; at least 32 rows per warp
    constexpr int kWarps = kRsThreads / 32;
    int64_t warps = (int64_t(g.m) + 31) / 32;
    const int64_t cap = int64_t(mode.num_sms) * kWarps;
    if (warps > cap) warps = cap;
    if (warps < 1) warps = 1;
    g.warps = static_cast<int32_t>(warps);
    const unsigned grid = static_cast<unsigned>((warps + kWarps - 1) / kWarps);
    g_last_kernel = "k_flop_rs (row streams, degree table in shared memory)";
    k_flop_rs<PRED><<<grid, kRsThreads, flop_rs_smem_bytes(k_rows), stream>>>(g, bdeg, k_rows, pred);
    return cudaGetLastError();
}

cudaError_t launch_flop_rows(const DevCsr& a, const uint16_t* bdeg, const int64_t* brpt, int64_t* flop,
                             long long* totals, cudaStream_t stream, const PredOut& pred, const FlopMode& mode,
                             const unsigned* escapes) {
    if (a.rows == 0) return cudaSuccess;
    RbArgs g;
    g.arpt = a.rpt;
    g.acol = a.col;
    g.brpt = brpt;
    g.m = a.rows;
    g.flop = flop;
    g.totals = totals;
    g.escapes = escapes;
    const bool smem = !mode.no_smem && flop_rb_smem_fits(mode.b_rows);
    // (row streams keep 32-bit offsets within a warp's entries)
    const bool rs_ok = a.nnz < (int64_t(1) << 31) - (int64_t(1) << 16);
    if (smem && rs_ok && (flop_rs_on() || !flop_rb_staged_fits(mode.b_rows))) {
        RsArgs r;
        r.arpt = a.rpt;
        r.acol = a.col;
        r.brpt = brpt;
        r.lo = a.base;
        r.hi = a.base + a.nnz;
        r.m = a.rows;
        r.flop = flop;
        r.totals = totals;
        r.escapes = escapes;
        r.k_rows = mode.b_rows;
        return pred.on() ? launch_rs<true>(r, bdeg, mode.b_rows, pred, mode, stream)
                         : launch_rs<false>(r, bdeg, mode.b_rows, pred, mode, stream);
    }
    if (smem && flop_rb_staged_fits(mode.b_rows))
        return pred.on() ? launch_rb<true, true>(g, bdeg, mode.b_rows, pred, mode, stream)
                         : launch_rb<true, false>(g, bdeg, mode.b_rows, pred, mode, stream);
    return pred.on() ? launch_rb<false, true>(g, bdeg, mode.b_rows, pred, mode, stream)
                     : launch_rb<false, false>(g, bdeg, mode.b_rows, pred, mode, stream);
}

cudaError_t launch_flop_fixup(const DevCsr& a, const FlopScratch& s, int64_t* flop, long long* totals,
                              cudaStream_t stream, const PredOut& pred) {
    const int64_t tiles = flop_tiles(a);
    if (tiles == 0) return cudaSuccess;
    constexpr int FB = 256;
    const unsigned gf = static_cast<unsigned>((tiles + FB - 1) / FB);
    if (pred.on())
        k_flop_fixup<FB, true><<<gf, FB, 0, stream>>>(s.tile_x, tiles, s.tile_carry, s.tile_total,
                                                      s.tile_max, flop, totals, pred);
    else
        k_flop_fixup<FB, false><<<gf, FB, 0, stream>>>(s.tile_x, tiles, s.tile_carry, s.tile_total,
                                                       s.tile_max, flop, totals, pred);
    return cudaGetLastError();
}

cudaError_t launch_flop(const DevCsr& a, const uint16_t* bdeg, const int64_t* brpt,
                        const FlopScratch& s, int64_t* flop, long long* totals,
                        cudaStream_t stream, const PredOut& pred, const FlopMode& mode) {
    const cudaError_t e = launch_flop_tiles(a, bdeg, brpt, s, flop, 0, flop_tiles(a), stream, pred, mode);
    if (e != cudaSuccess) return e;
    return launch_flop_fixup(a, s, flop, totals, stream, pred);
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

bool pattern_table_applies(const DevCsr& a, int32_t k_rows, bool rows_mode) {
    return !rows_mode && flop_rb_smem_fits(k_rows) && flop_rs_on() &&
           a.nnz < (int64_t(1) << 31) - (int64_t(1) << 16) && a.nnz >= kRsChunk;
}

cudaError_t launch_pattern_table(const DevCsr& a, const uint16_t* deg, int32_t k_rows, int num_sms, bool gather,
                                 long long* out, cudaStream_t stream) {
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_done.load(std::memory_order_acquire) & (1ull << (dev & 63)))) {
        cudaFuncSetAttribute(k_pattern_table<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(227 * 1024 - kSmemStatic));
        attr_done.fetch_or(1ull << (dev & 63), std::memory_order_release);
    }
    if (gather)
        k_pattern_table<true><<<num_sms, kRsThreads, flop_rs_smem_bytes(k_rows), stream>>>(a.col, a.base, a.nnz,
                                                                                           deg, k_rows, out);
    else
        k_pattern_table<false><<<num_sms, kRsThreads, 0, stream>>>(a.col, a.base, a.nnz, deg, k_rows, out);
    return cudaGetLastError();
}

}  // namespace spnnz_gpu
