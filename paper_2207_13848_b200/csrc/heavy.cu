// Heavy rows of the symbolic engine (FLOP > kBin5Max): exact distinct-column
// counts with every set operation in shared memory.
//
// A heavy row of C = A*B can have millions of products (config 5: up to
// 1.2 M, 84 M over 1 249 sampled rows) and its distinct set does not fit one
// SM.  A per-row global bitmap (2 MB at config 5, ~850 rows in flight)
// thrashes L2 into gigabytes of DRAM read-modify-write, so the columns are cut
// into ranges of W = 2^19 (a 64 KB shared bitmap) and each (row, range) is
// counted on chip.  Per batch of heavy rows:
//   0. prep / entries   unit (4096 products), entry and product offsets of
//                       every row; per entry its product prefix and B-row
//                       start; a unit -> (row, first entry) map;
//   1 < R <= 256 ranges (B.cols <= 2^27, the default path):
//   1. sort_units   each unit's products are enumerated, counting-sorted by
//                   range in shared memory and written back in place with the
//                   unit's R + 1 range starts; per-(row, range) totals;
//   2. plan_units   a task per (row, range); ranges above kTaskProducts split
//                   into unit groups sharing a merge slot; ranges of at most
//                   kSmallTaskProducts go to a separate list;
//   3. run_units    3 x 512-thread blocks per SM, one bitmap task each: the
//                   range is read as one slice per unit, each bit atomically
//                   OR-ed and the bits set first counted; split ranges OR
//                   their non-zero words into a global merge bitmap and count
//                   popc(word & ~old); the next task's descriptor and table
//                   entries are fetched while the current one runs;
//   4. run_small    small ranges: four 128-thread groups per block, each with
//                   a 4096-slot shared hash and its own named barrier;
//   R == 1 (B.cols <= 2^20): tasks are product slices read straight from the
//                   B rows (1024 threads, 128 KB bitmap, merge slots);
//   R > 256: count -> offsets -> place -> plan -> run over global buckets;
//   opt-in interval path (SPNNZ_HEAVY_INTERVALS=1, B rows sorted): a
//                   per-(entry, interval) boundary table replaces the product
//                   buffer (exact; slower at config 5).
// Every count is a set cardinality: exact and independent of bucketing, task
// boundaries and scheduling.
#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "symbolic_common.cuh"

namespace spnnz_gpu {
namespace {
using namespace sym;

#ifndef SPNNZ_HB
#define SPNNZ_HB 256
#endif
constexpr int kHB = SPNNZ_HB;             // block of the unit passes
constexpr int kHW = kHB / 32;             // warps per unit block
constexpr int kSpanShift = 20;            // R == 1: one span of <= 2^20 columns (128 KB)
#ifndef SPNNZ_SPAN_SHIFT
#define SPNNZ_SPAN_SHIFT 19
#endif
#ifndef SPNNZ_RUN_GRID
#define SPNNZ_RUN_GRID 3
#endif
constexpr int kTaskSpanShift = SPNNZ_SPAN_SHIFT;  // R > 1: task spans of <= 2^19 columns (64 KB)
constexpr int kPrivRanges = 256;          // per-warp histograms up to this R
constexpr int kMaxRanges = 4096;          // B.cols < 2^31 with W = 2^19
#ifndef SPNNZ_TASK_PRODUCTS
#define SPNNZ_TASK_PRODUCTS 131072
#endif
constexpr int64_t kTaskProducts = SPNNZ_TASK_PRODUCTS;
// A/B knob: bitmap inserts that read the word first and skip the atomic when
// the bit is already set (a duplicate product).  Measured slower (config 2
// symbolic 299 vs 282 us, where 57 % of the products are duplicates), so off.
#ifndef SPNNZ_BITMAP_TEST
#define SPNNZ_BITMAP_TEST 0
#endif
constexpr bool kTestFirst = SPNNZ_BITMAP_TEST != 0;
// A/B knob: the unit sort's range ranks from runs of equal ranges in lane
// order (0), __match_any_sync (1) or one ballot per range bit (2)
#ifndef SPNNZ_SORT_MATCH
#define SPNNZ_SORT_MATCH 1
#endif
#ifndef SPNNZ_SMALL_TASK
#define SPNNZ_SMALL_TASK 2048
#endif
constexpr int64_t kSmallTaskProducts = SPNNZ_SMALL_TASK;  // (A/B: 1024 / 512, see DESIGN)
#ifndef SPNNZ_RUN_U
#define SPNNZ_RUN_U 8
#endif
constexpr int kRunU = SPNNZ_RUN_U;
#ifndef SPNNZ_SORT_U
#define SPNNZ_SORT_U 8
#endif
constexpr int kSortU = SPNNZ_SORT_U;  // keys in flight per lane in the unit sort  // keys in flight per lane, R == 1 tasks (products straight from B)  // ranges this small go to k_heavy_run_small

struct HeavyTask {
    int32_t item;    // index in the batch
    int32_t slot;    // merge bitmap slot, or -1
    int32_t r0, r1;  // column ranges [r0, r1) (R > 1)
    int64_t a, b;    // R > 1: product-buffer span; R == 1: the item's product range
};
static_assert(sizeof(HeavyTask) == 32, "task layout");

// Shared bitmap inserts on a register-held window address (shared_window_reg):
// bit `off` of the bitmap at set_s.  The generic-pointer atomicOr re-derived
// the shared window -- and the task's column base -- for every key.
__device__ __forceinline__ void bit_set(uint32_t set_s, uint32_t off) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(set_s + ((off >> 3) & ~3u)), "r"(1u << (off & 31)) : "memory");
}
__device__ __forceinline__ int bit_set_new(uint32_t set_s, uint32_t off) {  // 1 if the bit was clear
    uint32_t old;
    asm volatile("atom.shared.or.b32 %0, [%1], %2;"
                 : "=r"(old) : "r"(set_s + ((off >> 3) & ~3u)), "r"(1u << (off & 31)) : "memory");
    return static_cast<int>(~(old >> (off & 31)) & 1u);
}
// Swizzled bit positions for the one-span bitmaps (R == 1, spans of >= 2^10
// bits): a warp's 32 keys are consecutive products of sorted B rows -- close
// columns -- and in the plain layout they pile onto a few words of a few
// banks (config 2: 13.9 M of the run kernel's 17.8 M shared wavefronts were
// bank conflicts).  Column offset o = low5 | mid5 << 5 | high << 10 goes to
// word low5 | high << 5 (its bank is the column's low five bits), bit mid5: a
// bijection of the span, so counts and merge slots are unchanged.
template <bool SWZ>
__device__ __forceinline__ void bit_set_l(uint32_t set_s, uint32_t off) {
    if (!SWZ) return bit_set(set_s, off);
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(set_s + (((off & 31u) | ((off >> 10) << 5)) << 2)),
                 "r"(1u << ((off >> 5) & 31u)) : "memory");
}
template <bool SWZ>
__device__ __forceinline__ int bit_set_new_l(uint32_t set_s, uint32_t off) {
    if (!SWZ) return bit_set_new(set_s, off);
    uint32_t old;
    asm volatile("atom.shared.or.b32 %0, [%1], %2;"
                 : "=r"(old) : "r"(set_s + (((off & 31u) | ((off >> 10) << 5)) << 2)), "r"(1u << ((off >> 5) & 31u))
                 : "memory");
    return static_cast<int>(~(old >> ((off >> 5) & 31u)) & 1u);
}
__device__ __forceinline__ int32_t opaque_reg(int32_t v) {
    asm volatile("" : "+r"(v));
    return v;
}

__device__ __forceinline__ const int32_t* heavy_list(const SymScratch& sc, int64_t first) {
    return sc.lists + int64_t(kHeavyBin) * sc.capacity + first;
}

// ---- 0a. batch bookkeeping: per item its units, entries, products,
// interval tasks and boundary-table cells, as exclusive prefixes (1 block)
#ifndef SPNNZ_PREP_BLOCK
#define SPNNZ_PREP_BLOCK 1024
#endif
constexpr int kPrepBlock = SPNNZ_PREP_BLOCK;

__global__ void __launch_bounds__(kPrepBlock) k_heavy_prep(SymArgs g, SymScratch sc, int64_t first,
                                                           int64_t count) {
    using Scan = cub::BlockScan<long long, kPrepBlock>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ long long s_carry[4];
    if (threadIdx.x < 4) s_carry[threadIdx.x] = 0;
    __syncthreads();
    const int32_t* list = heavy_list(sc, first);
    for (int64_t b = 0; b < count; b += kPrepBlock) {
        const int64_t i = b + threadIdx.x;
        long long x[4] = {0, 0, 0, 0};
        if (i < count) {
            const int32_t s = list[i];
            const int32_t rid = g.rows ? g.rows[s] : g.row_lo + s;
            const ItemRow it = item_row(g, s);
            const long long f = g.item_flop ? g.item_flop[s] : g.flop[rid - g.row_lo];
            const long long L = it.a1 - it.a0;
            x[0] = (f + kHeavyUnitProducts - 1) / kHeavyUnitProducts;  // units
            x[1] = L + 1;                                               // entries (+ end)
            x[2] = f;                                                   // products
            x[3] = (interval_geometry(g.bcols).count - 1) * L;          // boundary cells
        }
        long long ex[4], tot[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            Scan(tmp).ExclusiveSum(x[k], ex[k], tot[k]);
            __syncthreads();
        }
        if (i < count) {
            sc.heavy_unit_off[i] = s_carry[0] + ex[0];
            sc.heavy_eoff[i] = s_carry[1] + ex[1];
            sc.heavy_foff[i] = s_carry[2] + ex[2];
            if (sc.heavy_boff) sc.heavy_boff[i] = s_carry[3] + ex[3];
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int k = 0; k < 4; ++k) s_carry[k] += tot[k];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        sc.heavy_unit_off[count] = s_carry[0];
        sc.heavy_eoff[count] = s_carry[1];
        sc.heavy_foff[count] = s_carry[2];
        if (sc.heavy_boff) sc.heavy_boff[count] = s_carry[3];
        sc.heavy_meta[0] = s_carry[0];
        sc.heavy_meta[3] = 0;  // tasks
        sc.heavy_meta[4] = 0;  // merge slots
        sc.heavy_meta[7] = 0;  // interval-task cursor
        sc.heavy_meta[8] = 0;  // small tasks
        sc.heavy_meta[10] = 0;  // the bitmap runs' task ticket
        sc.heavy_meta[11] = 0;  // k_heavy_run_small's task ticket
    }
}

// ---- 0b. one block per item: product prefix over its entries, B-row starts.
// kEntV consecutive entries per thread, their loads issued together, so a
// row of up to kEntB * kEntV entries costs one dependent load chain (the
// walk of 256 entries per step made the longest heavy row the critical path:
// ~30 us whatever the number of heavy rows).
#ifndef SPNNZ_ENT_BLOCK
#define SPNNZ_ENT_BLOCK 512
#endif
constexpr int kEntB = SPNNZ_ENT_BLOCK, kEntV = 4;
__global__ void __launch_bounds__(kEntB) k_heavy_entries(SymArgs g, SymScratch sc, int64_t first) {
    using Scan = cub::BlockScan<long long, kEntB>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ long long s_carry;
    const int64_t i = blockIdx.x;
    const ItemRow it = item_row(g, heavy_list(sc, first)[i]);
    int64_t* ep = sc.heavy_epre + sc.heavy_eoff[i];
    int64_t* eb = sc.heavy_eb0 + sc.heavy_eoff[i];
    const int64_t L = it.a1 - it.a0;
    const int64_t ubase = sc.heavy_unit_off[i];
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < L; c0 += int64_t(kEntB) * kEntV) {
        const int64_t e0 = c0 + int64_t(threadIdx.x) * kEntV;
        int c[kEntV];
        long long d[kEntV];
        int64_t b0[kEntV];
#pragma unroll
        for (int k = 0; k < kEntV; ++k) c[k] = e0 + k < L ? __ldg(&g.a.col[it.a0 + e0 + k]) : -1;
#pragma unroll
        for (int k = 0; k < kEntV; ++k) {
            b0[k] = c[k] >= 0 ? __ldg(&g.brpt[c[k]]) : 0;
            d[k] = c[k] >= 0 ? __ldg(&g.brpt[c[k] + 1]) : 0;
        }
        long long sum = 0;
#pragma unroll
        for (int k = 0; k < kEntV; ++k) {
            d[k] -= b0[k];
            sum += d[k];
        }
        long long ex, tot;
        Scan(tmp).ExclusiveSum(sum, ex, tot);
        long long p = s_carry + ex;
#pragma unroll
        for (int k = 0; k < kEntV; ++k) {
            const int64_t e = e0 + k;
            if (e < L) {
                ep[e] = p;
                eb[e] = b0[k];
                if (sc.heavy_unit_item) {  // units whose first product is in this entry
                    for (long long u = (p + kHeavyUnitProducts - 1) / kHeavyUnitProducts;
                         u * kHeavyUnitProducts < p + d[k]; ++u) {
                        sc.heavy_unit_item[ubase + u] = static_cast<int32_t>(i);
                        sc.heavy_unit_e0[ubase + u] = static_cast<int32_t>(e);
                    }
                }
            }
            p += d[k];
        }
        __syncthreads();
        if (threadIdx.x == 0) s_carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) ep[L] = s_carry;
}

struct Unit {
    int64_t item;
    long long p0, p1;  // product window of the item
    int64_t e0;        // entry holding product p0, or -1 (unknown)
};

__device__ __forceinline__ Unit find_unit(const SymScratch& sc, int64_t count, long long u) {
    Unit r;
    if (sc.heavy_unit_item) {  // the unit map written by k_heavy_entries
        r.item = sc.heavy_unit_item[u];
        r.e0 = sc.heavy_unit_e0[u];
    } else {
        int64_t lo = 0, hi = count - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (sc.heavy_unit_off[mid] <= u) lo = mid; else hi = mid - 1;
        }
        r.item = lo;
        r.e0 = -1;
    }
    const long long ftot = sc.heavy_foff[r.item + 1] - sc.heavy_foff[r.item];
    r.p0 = (u - sc.heavy_unit_off[r.item]) * kHeavyUnitProducts;
    r.p1 = r.p0 + kHeavyUnitProducts < ftot ? r.p0 + kHeavyUnitProducts : ftot;
    return r;
}

// Every thread gets unit u (block-uniform call; the barrier also separates
// consecutive units' use of shared memory).
__device__ __forceinline__ Unit find_unit_block(const SymScratch& sc, int64_t count, long long u) {
    __shared__ Unit s_unit;
    __syncthreads();
    if (sc.heavy_unit_item) return find_unit(sc, count, u);
    if (threadIdx.x == 0) s_unit = find_unit(sc, count, u);
    __syncthreads();
    return s_unit;
}

// Block-wide walk over products [p0, p1) of heavy item `item` (p1 - p0 <
// 2^31): chunks of BLOCK entries are staged in shared memory with offsets
// relative to p0 (clamped to [0, p1 - p0], B-row starts shifted to match) so
// the per-product cursor works in 32-bit.  fn(keys, valid, q) with keys[u]
// = product p0 + q + 32 u.  e0: the entry holding product p0, or -1.
template <int BLOCK, int U = kUnroll, typename Fn>
__device__ __forceinline__ void item_products(const SymArgs& g, const SymScratch& sc,
                                              int64_t first, int64_t item, long long p0,
                                              long long p1, int* s_off, int64_t* s_b0, Fn&& fn,
                                              int64_t e0 = -1) {
    const ItemRow it = item_row(g, heavy_list(sc, first)[item]);
    const int64_t L = it.a1 - it.a0;
    const int64_t* ep = sc.heavy_epre + sc.heavy_eoff[item];
    const int64_t* eb = sc.heavy_eb0 + sc.heavy_eoff[item];
    const long long span = p1 - p0;
    __shared__ int64_t s_e0;
    if (e0 < 0) {
        __syncthreads();  // s_e0 of a previous call is consumed
        if (threadIdx.x == 0) {
            int64_t lo = 0, hi = L - 1;  // largest entry with ep[e] <= p0
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (ep[mid] <= p0) lo = mid; else hi = mid - 1;
            }
            s_e0 = lo;
        }
        __syncthreads();
        e0 = s_e0;
    }
    for (int64_t e = e0;;) {
        const int n = static_cast<int>(L - e < BLOCK ? L - e : BLOCK);
        __syncthreads();  // previous chunk fully consumed
        for (int i = threadIdx.x; i <= n; i += BLOCK) {
            const long long rel = ep[e + i] - p0;
            const long long cl = rel < 0 ? 0 : (rel > span ? span : rel);
            s_off[i] = static_cast<int>(cl);
            if (i < n) s_b0[i] = eb[e + i] + (cl - rel);
        }
        __syncthreads();
        chunk_products<BLOCK / 32, U>(s_off, s_b0, n, s_off[0], s_off[n], g.bcol, fn);
        const bool done = s_off[n] >= span || e + n >= L;
        if (done) break;
        e += n;
    }
    __syncthreads();
}

// ---- 1. per-unit histogram over column ranges, added to the bucket counts
__global__ void __launch_bounds__(kHB) k_heavy_count(SymArgs g, SymScratch sc, int64_t first,
                                                     int64_t count, int R, int wshift) {
    constexpr int NW = 1, RM = kMaxRanges;  // R > kPrivRanges: one shared histogram
    __shared__ int s_off[kHB + 1];
    __shared__ int64_t s_b0[kHB];
    __shared__ int s_hist[NW][RM];
    constexpr int w = 0;
    const long long units = sc.heavy_meta[0];
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        const Unit un = find_unit_block(sc, count, u);
        for (int k = threadIdx.x; k < NW * R; k += kHB) s_hist[k / R][k % R] = 0;
        item_products<kHB>(g, sc, first, un.item, un.p0, un.p1, s_off, s_b0,
                           [&](const int (&keys)[kUnroll], const bool (&valid)[kUnroll], long long) {
#pragma unroll
                               for (int k = 0; k < kUnroll; ++k)
                                   if (valid[k]) atomicAdd(&s_hist[w][keys[k] >> wshift], 1);
                           }, un.e0);
        long long* rc = sc.heavy_rc + un.item * R;
        for (int r = threadIdx.x; r < R; r += kHB) {
            int c = 0;
#pragma unroll
            for (int v = 0; v < NW; ++v) c += s_hist[v][r];
            if (c)
                atomicAdd(reinterpret_cast<unsigned long long*>(&rc[r]),
                          static_cast<unsigned long long>(c));
        }
    }
}

// ---- 2. bucket starts (exclusive prefix per item, placed at foff[item])
__global__ void k_heavy_offsets(SymScratch sc, int64_t count, int R) {
    const int64_t i = blockIdx.x;
    using Scan = cub::BlockScan<long long, 256>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ long long s_carry;
    if (threadIdx.x == 0) s_carry = sc.heavy_foff[i];
    __syncthreads();
    long long* rc = sc.heavy_rc + i * R;
    long long* cur = sc.heavy_cur + i * R;
    for (int r0 = 0; r0 < R; r0 += 256) {
        const int r = r0 + threadIdx.x;
        const long long c = r < R ? rc[r] : 0;
        long long ex, tot;
        Scan(tmp).ExclusiveSum(c, ex, tot);
        if (r < R) {
            rc[r] = s_carry + ex;
            cur[r] = s_carry + ex;
        }
        __syncthreads();
        if (threadIdx.x == 0) s_carry += tot;
        __syncthreads();
    }
}

// ---- 3. place: counting-sort each unit by range in shared memory, write the
// sorted runs to their bucket slices (coalesced)
__global__ void __launch_bounds__(kHB) k_heavy_place(SymArgs g, SymScratch sc, int64_t first,
                                                     int64_t count, int R, int wshift) {
    constexpr int NW = 1, RM = kMaxRanges;  // R > kPrivRanges: one shared histogram
    __shared__ int s_off[kHB + 1];
    __shared__ int64_t s_b0[kHB];
    // dynamic: dst_base[RM] (int64: bucket position of the unit's first key of
    //          range r, minus its sorted position) | keys_in[U] | keys_out[U] |
    //          hist[NW][RM] | offs[RM + 1]
    extern __shared__ int4 s_dyn_place[];
    long long* s_dst = reinterpret_cast<long long*>(s_dyn_place);
    int32_t* s_in = reinterpret_cast<int32_t*>(s_dst + RM);
    int32_t* s_out = s_in + kHeavyUnitProducts;
    int (*s_hist)[RM] = reinterpret_cast<int (*)[RM]>(s_out + kHeavyUnitProducts);
    int* s_offs = reinterpret_cast<int*>(s_hist + NW);
    constexpr int w = 0;
    const int lane = threadIdx.x & 31;
    const long long units = sc.heavy_meta[0];
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        const Unit un = find_unit_block(sc, count, u);
        for (int k = threadIdx.x; k < NW * R; k += kHB) s_hist[k / R][k % R] = 0;
        item_products<kHB>(g, sc, first, un.item, un.p0, un.p1, s_off, s_b0,
                           [&](const int (&keys)[kUnroll], const bool (&valid)[kUnroll],
                               long long q) {
#pragma unroll
                               for (int k = 0; k < kUnroll; ++k)
                                   if (valid[k]) s_in[q + 32 * k] = keys[k];
                           }, un.e0);
        const int n = static_cast<int>(un.p1 - un.p0);
        for (int i = threadIdx.x; i < n; i += kHB) atomicAdd(&s_hist[w][s_in[i] >> wshift], 1);
        __syncthreads();
        // per range: totals, per-warp offsets inside the range, bucket reservation
        long long* cur = sc.heavy_cur + un.item * R;
        for (int r = threadIdx.x; r < R; r += kHB) {
            int tot = 0;
#pragma unroll
            for (int v = 0; v < NW; ++v) {
                const int c = s_hist[v][r];
                s_hist[v][r] = tot;
                tot += c;
            }
            s_offs[r] = tot;
            s_dst[r] = tot ? static_cast<long long>(atomicAdd(
                                 reinterpret_cast<unsigned long long*>(&cur[r]),
                                 static_cast<unsigned long long>(tot)))
                           : 0;
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // exclusive scan of the R totals by warp 0
            const int per = (R + 31) / 32;
            const int r0 = lane * per, r1 = r0 + per < R ? r0 + per : R;
            int sum = 0;
            for (int r = r0; r < r1; ++r) sum += s_offs[r];
            int incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            int run = incl - sum;
            for (int r = r0; r < r1; ++r) {
                const int c = s_offs[r];
                s_offs[r] = run;
                s_dst[r] -= run;  // position i of range r goes to s_dst[r] + i
                run += c;
            }
            if (lane == 31) s_offs[R] = incl;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += kHB) {  // same thread <-> item mapping
            const int key = s_in[i];
            const int r = key >> wshift;
            s_out[s_offs[r] + atomicAdd(&s_hist[w][r], 1)] = key;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += kHB) {
            const int key = s_out[i];
            sc.heavy_pbuf[s_dst[key >> wshift] + i] = key;
        }
        __syncthreads();
    }
}

// ---- 3u. (1 < R <= kPrivRanges) sort each unit in place instead of count +
// place: the unit's products are counting-sorted by range and written back to
// the unit's own window of the product buffer, with its R + 1 range starts in
// heavy_utab; the per-(item, range) totals go to heavy_rc for the planner.  A
// task then reads range r as one slice per unit.
// A warp's 32 keys are consecutive products -- runs of one sorted B row -- so
// they fall in a few ranges: lanes of one range combine (warp_range_rank:
// one ballot per range bit) and their lowest lane takes the block's cursor
// for all of them, where per-lane atomics on the same counter serialised
// (63 M of the kernel's 88 M shared wavefronts were bank conflicts at config
// 5).  The rank within the range is kept beside the key; after the scan of
// the range totals each key is written straight to its final position.
// counters_s: the 32-bit shared-window address of the range counters (the
// generic-pointer atomicAdd re-derived the window for every key)
__device__ __forceinline__ int shared_add(uint32_t addr, int v) {
    int old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ int warp_range_rank(uint32_t counters_s, int bucket, bool valid, int nbits) {
    const int lane = threadIdx.x & 31;
#if SPNNZ_SORT_MATCH == 1
    unsigned peers = __match_any_sync(kFull, valid ? bucket : -1);
    if (!valid) peers = 0u;
    const int leader = peers ? __ffs(peers) - 1 : lane;
    int base = 0;
    if (valid && lane == leader) base = shared_add(counters_s + 4u * bucket, __popc(peers));
    base = __shfl_sync(kFull, base, leader);
    return base + __popc(peers & ((1u << lane) - 1));
#elif SPNNZ_SORT_MATCH == 2
    unsigned peers = __ballot_sync(kFull, valid);
    for (int b = 0; b < nbits; ++b) {
        const bool bit = (bucket >> b) & 1;
        const unsigned bal = __ballot_sync(kFull, bit);
        peers &= bit ? bal : ~bal;
    }
    const int leader = peers ? __ffs(peers) - 1 : lane;
    int base = 0;
    if (valid && lane == leader) base = shared_add(counters_s + 4u * bucket, __popc(peers));
    base = __shfl_sync(kFull, base, leader);
    return base + __popc(peers & ((1u << lane) - 1));
#else
    // runs of equal ranges in lane order (the keys are sorted within a B
    // row): each run's first lane takes the cursor for the run
    (void)nbits;
    const int prev = __shfl_up_sync(kFull, bucket, 1);
    const unsigned vmask = __ballot_sync(kFull, valid);
    const unsigned heads = __ballot_sync(kFull, valid && (lane == 0 || prev != bucket)) | ~vmask;
    const unsigned le = 0xffffffffu >> (31 - lane);       // lanes <= lane
    const int head = 31 - __clz(heads & le);               // this lane's run head
    const unsigned after = heads & ~le;                    // heads (or invalid lanes) above the lane
    const int next = after ? __ffs(after) - 1 : 32;
    int base = 0;
    if (valid && head == lane) base = shared_add(counters_s + 4u * bucket, next - lane);
    base = __shfl_sync(kFull, base, head);
    return base + lane - head;
#endif
}

__global__ void __launch_bounds__(kHB, 1536 / kHB) k_heavy_sort_units(SymArgs g, SymScratch sc, int64_t first,
                                                          int64_t count, int R, int wshift) {
    __shared__ int s_off[kHB + 1];
    __shared__ int64_t s_b0[kHB];
    // dynamic: keys[U] | ranks[U] | hist[R] (kHW * R reserved) | offs[R + 1]
    extern __shared__ int4 s_dyn_sort[];
    int32_t* s_in = reinterpret_cast<int32_t*>(s_dyn_sort);
    int32_t* s_rank = s_in + kHeavyUnitProducts;
    int* s_hist = s_rank + kHeavyUnitProducts;
    int* s_offs = s_hist + kHW * R;
    const int lane = threadIdx.x & 31;
    const int nbits = 32 - __clz(R - 1);
    // shared-window addresses held in registers (opaque to the compiler, which
    // otherwise re-derives the window -- S2UR SR_CgaCtaId + three uniform
    // instructions -- at every store and atomic of the rank loop)
    uint32_t in_s = static_cast<uint32_t>(__cvta_generic_to_shared(s_in));
    uint32_t hist_s = static_cast<uint32_t>(__cvta_generic_to_shared(s_hist));
    asm volatile("" : "+r"(in_s), "+r"(hist_s));
    const long long units = sc.heavy_meta[0];
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        const Unit un = find_unit_block(sc, count, u);
        for (int k = threadIdx.x; k < R; k += kHB) s_hist[k] = 0;
        // (item_products starts with a barrier: the counters are zero before
        // the first rank is taken)
        item_products<kHB, kSortU>(g, sc, first, un.item, un.p0, un.p1, s_off, s_b0,
                           [&](const int (&keys)[kSortU], const bool (&valid)[kSortU],
                               long long q) {
#pragma unroll
                               const uint32_t at = in_s + 4u * static_cast<uint32_t>(q);
                               for (int k = 0; k < kSortU; ++k) {
                                   const int rk = warp_range_rank(hist_s, keys[k] >> wshift, valid[k], nbits);
                                   if (valid[k]) {  // s_in[q + 32 k] = key, s_rank[q + 32 k] = rank
                                       asm volatile("st.shared.b32 [%0], %1;" ::"r"(at + 128u * k), "r"(keys[k]) : "memory");
                                       asm volatile("st.shared.b32 [%0], %1;" ::"r"(at + 128u * k + static_cast<uint32_t>(4 * kHeavyUnitProducts)), "r"(rk) : "memory");
                                   }
                               }
                           }, un.e0);
        const int n = static_cast<int>(un.p1 - un.p0);
        // range totals -> the planner's per-(item, range) counts
        long long* rc = sc.heavy_rc + un.item * R;
        for (int r = threadIdx.x; r < R; r += kHB)
            if (s_hist[r]) atomicAdd(reinterpret_cast<unsigned long long*>(&rc[r]), static_cast<unsigned long long>(s_hist[r]));
        if (threadIdx.x < 32) {  // exclusive scan of the R totals by warp 0
            const int per = (R + 31) / 32;
            const int r0 = lane * per, r1 = r0 + per < R ? r0 + per : R;
            int sum = 0;
            for (int r = r0; r < r1; ++r) sum += s_hist[r];
            const int incl = warp_incl_scan(sum);
            int run = incl - sum;
            for (int r = r0; r < r1; ++r) {
                s_offs[r] = run;
                run += s_hist[r];
            }
            if (lane == 31) s_offs[R] = incl;
        }
        __syncthreads();
        int32_t* dst = sc.heavy_pbuf + sc.heavy_foff[un.item] + un.p0;
        for (int i = threadIdx.x; i < n; i += kHB) {
            const int key = s_in[i];
            dst[s_offs[key >> wshift] + s_rank[i]] = key;
        }
        int32_t* tab = sc.heavy_utab + u * (R + 1);
        for (int r = threadIdx.x; r <= R; r += kHB) tab[r] = s_offs[r];
    }
}

// Unit-sorted tasks: one block per item, one thread per range; a range above
// kTaskProducts products is split into groups of the item's units that share
// a merge slot.
__global__ void __launch_bounds__(kPrivRanges) k_heavy_plan_units(SymScratch sc, int64_t count, int R,
                                                                  int64_t task_cap) {
    using Scan = cub::BlockScan<int, kPrivRanges>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ long long s_base;
    const int64_t i = blockIdx.x;
    const int r = threadIdx.x;
    const long long nu = sc.heavy_unit_off[i + 1] - sc.heavy_unit_off[i];
    const long long cnt = r < R ? sc.heavy_rc[i * R + r] : 0;
    const bool small = cnt > 0 && cnt <= kSmallTaskProducts;
    long long p = (cnt + kTaskProducts - 1) / kTaskProducts;
    const int parts = small ? 0 : static_cast<int>(p < nu ? p : nu);
    int excl, total;
    Scan(tmp).ExclusiveSum(parts, excl, total);
    if (threadIdx.x == 0)
        s_base = static_cast<long long>(atomicAdd(reinterpret_cast<unsigned long long*>(&sc.heavy_meta[3]),
                                                  static_cast<unsigned long long>(total)));
    __shared__ long long s_cnt[kPrivRanges];
    __shared__ int s_g0[kPrivRanges], s_g1[kPrivRanges];
    s_cnt[r] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        // small ranges: a list of their own, filled from the end of the array;
        // consecutive small (and empty) ranges share one task up to
        // kSmallTaskProducts products (fewer tasks each reading every unit's
        // table; the 4096-slot hash holds any 2048 products at load <= 1/2)
        int ng = 0;
        const auto emit_small = [&](int r0, int r1) {
            s_g0[ng] = r0;
            s_g1[ng++] = r1;
        };
        int g0 = 0;
        long long gsum = 0;
        for (int q = 0; q < R; ++q) {
            const long long c = s_cnt[q];
            if (c > kSmallTaskProducts) {  // a bitmap task: closes the group
                if (gsum > 0) emit_small(g0, q);
                g0 = q + 1;
                gsum = 0;
                continue;
            }
            if (gsum > 0 && gsum + c > kSmallTaskProducts) {
                emit_small(g0, q);
                g0 = q;
                gsum = 0;
            }
            gsum += c;
        }
        if (gsum > 0) emit_small(g0, R);
        // one reservation per item for its groups
        const long long k0 = ng ? static_cast<long long>(atomicAdd(
                                      reinterpret_cast<unsigned long long*>(&sc.heavy_meta[8]),
                                      static_cast<unsigned long long>(ng)))
                                : 0;
        for (int q = 0; q < ng; ++q)
            reinterpret_cast<HeavyTask*>(sc.heavy_tasks)[task_cap - 1 - (k0 + q)] =
                HeavyTask{static_cast<int32_t>(i), -1, s_g0[q], s_g1[q], 0, nu};
    }
    __syncthreads();
    if (s_base + total + sc.heavy_meta[8] > task_cap) __trap();  // host sizes task_cap to heavy_task_bound()
    if (parts > 0) {
        const int32_t slot = parts > 1 ? static_cast<int32_t>(atomicAdd(
                                             reinterpret_cast<unsigned long long*>(&sc.heavy_meta[4]), 1ULL))
                                       : -1;
        if (slot >= 0) sc.heavy_slot_item[slot] = static_cast<int32_t>(i);
        HeavyTask* out = reinterpret_cast<HeavyTask*>(sc.heavy_tasks) + s_base + excl;
        for (int q = 0; q < parts; ++q)
            out[q] = HeavyTask{static_cast<int32_t>(i), slot, r, r + 1, nu * q / parts, nu * (q + 1) / parts};
    }
}

// ---- 4. tasks
// R > 1: one block per item, one thread per aligned span.
__global__ void __launch_bounds__(128) k_heavy_plan(SymScratch sc, int64_t count, int R,
                                                    int wshift, int64_t task_cap) {
    using Scan = cub::BlockScan<int, 128>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ long long s_base;
    const int64_t i = blockIdx.x;
    const int per_span = 1 << (kTaskSpanShift - wshift);
    const int S = (R + per_span - 1) / per_span;
    const long long* rc = sc.heavy_rc + i * R;
    const long long end = sc.heavy_foff[i + 1];
    HeavyTask* tasks = reinterpret_cast<HeavyTask*>(sc.heavy_tasks);
    for (int s0 = 0; s0 < S; s0 += 128) {
        const int sp = s0 + threadIdx.x;
        const int r0 = sp * per_span, r1 = r0 + per_span < R ? r0 + per_span : R;
        long long a = 0, b = 0;
        int parts = 0;
        if (sp < S) {
            a = rc[r0];
            b = r1 < R ? rc[r1] : end;
            parts = static_cast<int>((b - a + kTaskProducts - 1) / kTaskProducts);
        }
        int excl, total;
        Scan(tmp).ExclusiveSum(parts, excl, total);
        if (threadIdx.x == 0)
            s_base = static_cast<long long>(atomicAdd(
                reinterpret_cast<unsigned long long*>(&sc.heavy_meta[3]),
                static_cast<unsigned long long>(total)));
        __syncthreads();
        if (s_base + total > task_cap) __trap();  // host sizes task_cap to heavy_task_bound()
        if (parts > 0) {
            const int32_t slot = parts > 1 ? static_cast<int32_t>(atomicAdd(
                                                 reinterpret_cast<unsigned long long*>(&sc.heavy_meta[4]), 1ULL))
                                           : -1;
            if (slot >= 0) sc.heavy_slot_item[slot] = static_cast<int32_t>(i);
            HeavyTask* out = tasks + s_base + excl;
            for (int q = 0; q < parts; ++q) {
                const long long p = a + q * kTaskProducts;
                out[q] = HeavyTask{static_cast<int32_t>(i), slot, r0, r1, p,
                                   p + kTaskProducts < b ? p + kTaskProducts : b};
            }
        }
        __syncthreads();
    }
}

// R == 1: one thread per item, parts of its product range.
__global__ void k_heavy_tasks_r1(SymScratch sc, int64_t count, int64_t task_cap) {
    const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (i >= count) return;
    const long long f = sc.heavy_foff[i + 1] - sc.heavy_foff[i];
    const long long parts = (f + kTaskProducts - 1) / kTaskProducts;
    if (parts == 0) return;
    const long long base = static_cast<long long>(atomicAdd(
        reinterpret_cast<unsigned long long*>(&sc.heavy_meta[3]), static_cast<unsigned long long>(parts)));
    if (base + parts > task_cap) __trap();
    const int32_t slot = parts > 1 ? static_cast<int32_t>(atomicAdd(
                                         reinterpret_cast<unsigned long long*>(&sc.heavy_meta[4]), 1ULL))
                                   : -1;
    if (slot >= 0) sc.heavy_slot_item[slot] = static_cast<int32_t>(i);
    HeavyTask* out = reinterpret_cast<HeavyTask*>(sc.heavy_tasks) + base;
    for (long long q = 0; q < parts; ++q) {
        const long long a = q * kTaskProducts;
        out[q] = HeavyTask{static_cast<int32_t>(i), slot, 0, 1, a, a + kTaskProducts < f ? a + kTaskProducts : f};
    }
}

// ORs a task's shared bitmap into its merge slot: non-returning reductions
// (red.global.or, ~1.6x the returning atomics' rate in L2, and no thread
// waits for a result); the slot's bits are counted once, after every task
// that shares it has merged (k_heavy_slot_count).  (Counting each task's
// first-set bits needed the returning atomic per word: at config 2 the largest
// rows split into ~30 tasks, 32 K words each.)
template <int BLOCK>
__device__ __forceinline__ void merge_words(const uint32_t* s_set, uint32_t* gbm, int32_t words) {
    for (int k = threadIdx.x; k < words; k += BLOCK) {
        const uint32_t w = s_set[k];
        if (w) asm volatile("red.global.or.b32 [%0], %1;" ::"l"(gbm + k), "r"(w) : "memory");
    }
}

// The used merge slots, cut into parts of kSlotPart words, one part per
// block at a time: the distinct columns its tasks found together (a partial
// count per part, added to the slot's item and to the total), the words
// zeroed on the way (the pool stays all-zero between calls).
constexpr int kSlotBlock = 256;
constexpr int64_t kSlotPart = 4096;  // words per part: 4 uint4 per thread
__global__ void __launch_bounds__(kSlotBlock) k_heavy_slot_count(SymArgs g, SymScratch sc, int64_t first,
                                                                 int64_t slot_words) {
    __shared__ long long s_red[kSlotBlock / 32];
    const long long used = sc.heavy_meta[4];
    const int32_t* list = heavy_list(sc, first);
    const int64_t parts = (slot_words + kSlotPart - 1) / kSlotPart;
    for (long long it = blockIdx.x; it < used * parts; it += gridDim.x) {
        const long long sl = it / parts;
        const int64_t w0 = (it % parts) * kSlotPart;
        const int64_t w1 = w0 + kSlotPart < slot_words ? w0 + kSlotPart : slot_words;
        uint32_t* w = sc.pool + sl * slot_words;
        long long c = 0;
        if (((w1 - w0) & 3) == 0 && (w0 & 3) == 0) {
            uint4* v4 = reinterpret_cast<uint4*>(w + w0);
            const int n4 = static_cast<int>((w1 - w0) >> 2);
            uint4 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int q = threadIdx.x + k * kSlotBlock;
                v[k] = q < n4 ? v4[q] : make_uint4(0u, 0u, 0u, 0u);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int q = threadIdx.x + k * kSlotBlock;
                if (q < n4) {
                    c += __popc(v[k].x) + __popc(v[k].y) + __popc(v[k].z) + __popc(v[k].w);
                    v4[q] = make_uint4(0u, 0u, 0u, 0u);
                }
            }
        } else {
            for (int64_t k = w0 + threadIdx.x; k < w1; k += kSlotBlock) {
                c += __popc(w[k]);
                w[k] = 0u;
            }
        }
        const long long tot = block_sum_ll<kSlotBlock>(c, s_red);
        if (threadIdx.x == 0 && tot) {
            if (g.out)
                atomicAdd(reinterpret_cast<unsigned long long*>(&g.out[list[sc.heavy_slot_item[sl]]]),
                          static_cast<unsigned long long>(tot));
            atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[g.total_slot]),
                      static_cast<unsigned long long>(tot));
        }
        __syncthreads();
    }
}

// ---- 5. run the tasks: one block per task, a shared bitmap over the span,
// kept all-zero between tasks.
// MODE: kRunItem (R == 1) products straight from the B rows; kRunBuckets the
// task's contiguous bucket span (unit-sorted buckets: k_heavy_run_units).
constexpr int kRunItem = 0, kRunBuckets = 1;

template <int kRunBlock, int MODE, bool SWZ = false>
__global__ void __launch_bounds__(kRunBlock) k_heavy_run(SymArgs g, SymScratch sc, int64_t first,
                                                         int R, int wshift, int32_t slot_words) {
    static_assert(!SWZ || MODE == kRunItem, "swizzled bitmaps: the one-span (R == 1) tasks");
    extern __shared__ int4 s_dyn[];
    uint32_t* s_set = reinterpret_cast<uint32_t*>(s_dyn);
    __shared__ int s_off[kRunBlock + 1];
    __shared__ int64_t s_b0[kRunBlock];
    __shared__ HeavyTask s_task;
    const HeavyTask* tasks = reinterpret_cast<const HeavyTask*>(sc.heavy_tasks);
    const long long ntask = sc.heavy_meta[3];
    const int32_t* list = heavy_list(sc, first);
    const int lane = threadIdx.x & 31;
    const int32_t max_words = R > 1 ? (1 << (kTaskSpanShift - 5))
                              : SWZ ? slot_words  // every word of the 2^wshift-bit span
                                    : static_cast<int32_t>((int64_t(g.bcols) + 31) / 32);
    for (int k = threadIdx.x; k < max_words; k += kRunBlock) s_set[k] = 0u;
    const uint32_t set_s = shared_window_reg(s_set);
    long long acc = 0;
    // tasks by ticket (a few hundred atomics): a block that starts late --
    // its SM still busy with a tier kernel -- takes fewer instead of holding
    // a fixed share back
    __shared__ long long s_ti;
    for (;;) {
        __syncthreads();  // previous task's clear is complete
        if (threadIdx.x == 0) {
            s_ti = static_cast<long long>(atomicAdd(reinterpret_cast<unsigned long long*>(&sc.heavy_meta[10]), 1ULL));
            if (s_ti < ntask) s_task = tasks[s_ti];
        }
        __syncthreads();
        if (s_ti >= ntask) break;
        const HeavyTask t = s_task;
        const int32_t col_base = opaque_reg(R > 1 ? (t.r0 << wshift) : 0);
        const int32_t words = R > 1 ? ((t.r1 - t.r0) << (wshift - 5)) : max_words;
        int cnt = 0;
        // a task that shares its span with others (merge slot) counts at the
        // merge, so its inserts need no return value (no wait on the atomic)
        const bool merged = t.slot >= 0;
        auto insert = [&](const auto& keys, const auto& valid, long long) {
            constexpr int UU = static_cast<int>(sizeof(valid) / sizeof(valid[0]));
            if (merged) {
#pragma unroll
                for (int u = 0; u < UU; ++u)
                    if (valid[u]) {
                        const uint32_t off = static_cast<uint32_t>(keys[u] - col_base);
                    SPNNZ_ASSERT((off >> 5) < static_cast<uint32_t>(words));
                        if (SWZ || !kTestFirst || !(s_set[off >> 5] & (1u << (off & 31)))) bit_set_l<SWZ>(set_s, off);
                    }
                return;
            }
#pragma unroll
            for (int u = 0; u < UU; ++u)
                if (valid[u]) {
                    const uint32_t off = static_cast<uint32_t>(keys[u] - col_base);
                    SPNNZ_ASSERT((off >> 5) < static_cast<uint32_t>(words));
                    if (SWZ || !kTestFirst || !(s_set[off >> 5] & (1u << (off & 31)))) cnt += bit_set_new_l<SWZ>(set_s, off);
                }
        };
        // the span's keys: 16-byte vectors over the aligned body, two vectors
        // per thread in flight; the unaligned head and tail (< 4 keys each)
        // go to the first threads
        auto contiguous = [&](auto&& fn) {
            long long a4 = (t.a + 3) & ~3LL;
            if (a4 > t.b) a4 = t.b;
            const long long n4 = (t.b - a4) >> 2, b4 = a4 + 4 * n4;
            const int head = static_cast<int>(a4 - t.a), tail = static_cast<int>(t.b - b4);
            if (threadIdx.x < head + tail) {
                const long long q = threadIdx.x < head ? t.a + threadIdx.x : b4 + (threadIdx.x - head);
                const int keys[kUnroll] = {__ldg(&sc.heavy_pbuf[q]), 0, 0, 0};
                const bool valid[kUnroll] = {true, false, false, false};
                fn(keys, valid, 0);
            }
            const int4* v = reinterpret_cast<const int4*>(sc.heavy_pbuf + a4);
            for (long long i = threadIdx.x; i < n4; i += 2 * kRunBlock) {
                const bool two = i + kRunBlock < n4;
                const int4 x = __ldg(v + i);
                const int4 y = two ? __ldg(v + i + kRunBlock) : make_int4(0, 0, 0, 0);
                const bool all[kUnroll] = {true, true, true, true};
                const int kx[kUnroll] = {x.x, x.y, x.z, x.w};
                fn(kx, all, 0);
                if (two) {
                    const int ky[kUnroll] = {y.x, y.y, y.z, y.w};
                    fn(ky, all, 0);
                }
            }
        };
        if constexpr (MODE == kRunBuckets) {
            contiguous(insert);
        } else {
            item_products<kRunBlock, kRunU>(g, sc, first, t.item, t.a, t.b, s_off, s_b0, insert);
        }
        __syncthreads();  // every insert is done
        if (t.slot >= 0) {
            // span shared by several tasks: the bits this task adds first
            cnt = 0;
            uint32_t* gbm = sc.pool + int64_t(t.slot) * slot_words;
            merge_words<kRunBlock>(s_set, gbm, words);
            cnt = 0;  // the slot's bits are counted once all its tasks are in (k_heavy_slot_count)
            __syncthreads();  // the merge scan has read the bitmap
        }
        cnt = static_cast<int>(warp_sum_ll(cnt));
        if (lane == 0 && cnt) {
            if (g.out)
                atomicAdd(reinterpret_cast<unsigned long long*>(&g.out[list[t.item]]),
                          static_cast<unsigned long long>(cnt));
            acc += cnt;
        }
        // back to all-zero: re-walk the keys of a sparse span, else clear
        if (MODE == kRunBuckets && (t.b - t.a) * 8 < words) {
            contiguous([&](const int (&keys)[kUnroll], const bool (&valid)[kUnroll], long long) {
#pragma unroll
                for (int v = 0; v < kUnroll; ++v)
                    if (valid[v]) s_set[static_cast<uint32_t>(keys[v] - col_base) >> 5] = 0u;
            });
        } else {
            uint4* s4 = reinterpret_cast<uint4*>(s_set);
            for (int k = threadIdx.x; k < (words >> 2); k += kRunBlock) s4[k] = make_uint4(0u, 0u, 0u, 0u);
            for (int k = (words & ~3) + threadIdx.x; k < words; k += kRunBlock) s_set[k] = 0u;
        }
    }
    if (lane == 0 && acc)
        atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[g.total_slot]),
                  static_cast<unsigned long long>(acc));
}

// ---- 5u. run for unit-sorted buckets, software-pipelined across tasks:
// while task i's products are walked, the descriptor and the unit-table
// entries of the block's next task are already in flight, so a task costs
// one global round trip less.  Tasks with more than kRunBlock units stage
// their slices in rounds (no prefetch).
#ifndef SPNNZ_UNITS_SWZ
#define SPNNZ_UNITS_SWZ 0
#endif
constexpr bool kUnitsSwz = SPNNZ_UNITS_SWZ != 0;  // A/B: the swizzled layout for the unit-sorted bitmap tasks
template <int kRunBlock>
__global__ void __launch_bounds__(kRunBlock, 3) k_heavy_run_units(SymArgs g, SymScratch sc, int64_t first,
                                                               int R, int wshift, int32_t slot_words) {
    extern __shared__ int4 s_dyn_ru[];
    uint32_t* s_set = reinterpret_cast<uint32_t*>(s_dyn_ru);
    using Scan = cub::BlockScan<int, kRunBlock>;
    __shared__ typename Scan::TempStorage s_scan;
    __shared__ int s_off[kRunBlock + 1];
    __shared__ int64_t s_b0[kRunBlock];
    const HeavyTask* tasks = reinterpret_cast<const HeavyTask*>(sc.heavy_tasks);
    const long long ntask = sc.heavy_meta[3];
    const int32_t* list = heavy_list(sc, first);
    const int lane = threadIdx.x & 31;
    constexpr int32_t kWords = 1 << (kTaskSpanShift - 5);
    for (int k = threadIdx.x; k < kWords; k += kRunBlock) s_set[k] = 0u;
    const uint32_t set_s = shared_window_reg(s_set);
    // unit-table entries of task t for this thread's unit (first round only)
    auto fetch = [&](const HeavyTask& t, int& lo, int& hi) {
        lo = hi = 0;
        if (threadIdx.x < t.b - t.a) {
            const int32_t* tab = sc.heavy_utab + (sc.heavy_unit_off[t.item] + t.a + threadIdx.x) * (R + 1);
            lo = tab[t.r0];
            hi = tab[t.r1];
        }
    };
    long long acc = 0;
    // tasks by ticket (as k_heavy_run); the next ticket and its descriptor
    // are taken while the current task runs
    __shared__ long long s_tk;
    const auto ticket = [&]() -> long long {
        __syncthreads();
        if (threadIdx.x == 0)
            s_tk = static_cast<long long>(atomicAdd(reinterpret_cast<unsigned long long*>(&sc.heavy_meta[10]), 1ULL));
        __syncthreads();
        return s_tk;
    };
    long long ti = ticket();
    HeavyTask tn{};
    int nlo = 0, nhi = 0;
    if (ti < ntask) {
        tn = tasks[ti];
        fetch(tn, nlo, nhi);
    }
    while (ti < ntask) {
        const HeavyTask t = tn;
        int lo = nlo, hi = nhi;
        const long long tj = ticket();
        if (tj < ntask) tn = tasks[tj];  // in flight during this task
        const int32_t col_base = opaque_reg(t.r0 << wshift);
        const int32_t words = (t.r1 - t.r0) << (wshift - 5);
        const long long pbase = sc.heavy_foff[t.item];
        int cnt = 0;
        auto insert = [&](const int (&keys)[kUnroll], const bool (&valid)[kUnroll], long long) {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
                if (valid[u]) {
                    const uint32_t off = static_cast<uint32_t>(keys[u] - col_base);
                    SPNNZ_ASSERT((off >> 5) < static_cast<uint32_t>(words));
                    if (kUnitsSwz || !kTestFirst || !(s_set[off >> 5] & (1u << (off & 31)))) cnt += bit_set_new_l<kUnitsSwz>(set_s, off);
                }
        };
        for (long long u0 = t.a; u0 < t.b; u0 += kRunBlock) {
            const int n = static_cast<int>(t.b - u0 < kRunBlock ? t.b - u0 : kRunBlock);
            if (u0 != t.a) {  // later rounds of a task with many units
                lo = hi = 0;
                if (threadIdx.x < n) {
                    const int32_t* tab = sc.heavy_utab + (sc.heavy_unit_off[t.item] + u0 + threadIdx.x) * (R + 1);
                    lo = tab[t.r0];
                    hi = tab[t.r1];
                }
            }
            int ex, tot;
            __syncthreads();  // the previous round / task is done with s_off, s_b0, s_set
            Scan(s_scan).ExclusiveSum(hi - lo, ex, tot);
            if (threadIdx.x < n) {
                s_off[threadIdx.x] = ex;
                s_b0[threadIdx.x] = pbase + (u0 + threadIdx.x) * kHeavyUnitProducts + lo;
            }
            if (threadIdx.x == 0) s_off[n] = tot;
            __syncthreads();
            if (u0 + kRunBlock >= t.b && tj < ntask) fetch(tn, nlo, nhi);  // next task's table, in flight
            chunk_products<kRunBlock / 32>(s_off, s_b0, n, 0, tot, sc.heavy_pbuf, insert);
        }
        __syncthreads();  // every insert is done
        if (t.slot >= 0) {
            // span shared by several tasks: the bits this task adds first
            cnt = 0;
            uint32_t* gbm = sc.pool + int64_t(t.slot) * slot_words;
            merge_words<kRunBlock>(s_set, gbm, words);
            cnt = 0;  // the slot's bits are counted once all its tasks are in (k_heavy_slot_count)
            __syncthreads();  // the merge scan has read the bitmap
        }
        cnt = static_cast<int>(warp_sum_ll(cnt));
        if (lane == 0 && cnt) {
            if (g.out)
                atomicAdd(reinterpret_cast<unsigned long long*>(&g.out[list[t.item]]),
                          static_cast<unsigned long long>(cnt));
            acc += cnt;
        }
        uint4* s4 = reinterpret_cast<uint4*>(s_set);
        for (int k = threadIdx.x; k < (words >> 2); k += kRunBlock) s4[k] = make_uint4(0u, 0u, 0u, 0u);
        ti = tj;
    }
    if (lane == 0 && acc)
        atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[g.total_slot]),
                  static_cast<unsigned long long>(acc));
}

// ---- 5s. small unit-sorted ranges (<= kSmallTaskProducts products): a
// 512-thread block is four independent 128-thread groups, each with a
// 4096-slot shared hash and its own named barrier, so an SM keeps twelve
// small tasks in flight instead of three bitmap tasks.
#ifndef SPNNZ_SMALL_GROUPS
#define SPNNZ_SMALL_GROUPS 4
#endif
#ifndef SPNNZ_SMALL_SLOTS
#define SPNNZ_SMALL_SLOTS 4096
#endif
constexpr int kSG = 128, kSGroups = SPNNZ_SMALL_GROUPS, kSSlots = SPNNZ_SMALL_SLOTS;
static_assert(kSSlots >= 2 * kSmallTaskProducts, "small-range table load <= 1/2");
constexpr int kSmallGrab = 2;  // small tasks per ticket

__device__ __forceinline__ void group_sync(int grp) {
    asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "r"(kSG) : "memory");
}

__global__ void __launch_bounds__(kSG * kSGroups, 3) k_heavy_run_small(SymArgs g, SymScratch sc, int64_t first,
                                                                       int R) {
    extern __shared__ int4 s_dyn_rs[];
    const int grp = threadIdx.x / kSG, gt = threadIdx.x % kSG, gw = gt >> 5, lane = threadIdx.x & 31;
    int* table = reinterpret_cast<int*>(s_dyn_rs) + grp * kSSlots;
    const uint32_t table_s = shared_window_reg(table);
    __shared__ int s_off[kSGroups][kSG + 1];
    __shared__ int64_t s_b0[kSGroups][kSG];
    __shared__ int s_wt[kSGroups][kSG / 32];
    const HeavyTask* tasks = reinterpret_cast<const HeavyTask*>(sc.heavy_tasks) + sc.heavy_task_cap - 1;
    const long long ntask = sc.heavy_meta[8];
    const int32_t* list = heavy_list(sc, first);
    long long acc = 0;
    // tasks by ticket, kSmallGrab per atomic (thousands of small tasks: one
    // counter, a few thousand atomics)
    __shared__ long long s_tk[kSGroups];
    long long tk = 0, tk_end = 0;
    for (;;) {
        if (tk == tk_end) {
            group_sync(grp);
            if (gt == 0)
                s_tk[grp] = static_cast<long long>(
                    atomicAdd(reinterpret_cast<unsigned long long*>(&sc.heavy_meta[11]), static_cast<unsigned long long>(kSmallGrab)));
            group_sync(grp);
            tk = s_tk[grp];
            tk_end = tk + kSmallGrab;
        }
        if (tk >= ntask) break;
        const long long ti = tk++;
        const HeavyTask t = *(tasks - ti);
        hash_clear(table, kSSlots, gt, kSG);
        const long long ubase = sc.heavy_unit_off[t.item];
        const long long pbase = sc.heavy_foff[t.item];
        int cnt = 0;
        for (long long u0 = t.a; u0 < t.b; u0 += kSG) {
            const int n = static_cast<int>(t.b - u0 < kSG ? t.b - u0 : kSG);
            int len = 0;
            int64_t start = 0;
            if (gt < n) {
                const long long u = u0 + gt;
                const int32_t* tab = sc.heavy_utab + (ubase + u) * (R + 1);
                const int lo = tab[t.r0];
                len = tab[t.r1] - lo;
                start = pbase + u * kHeavyUnitProducts + lo;
            }
            const int incl = warp_incl_scan(len);
            group_sync(grp);  // the previous round's walk is done with s_off / s_b0
            if (lane == 31) s_wt[grp][gw] = incl;
            group_sync(grp);
            int before = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < kSG / 32; ++w) {
                const int v = s_wt[grp][w];
                before += w < gw ? v : 0;
                tot += v;
            }
            if (gt < n) {
                s_off[grp][gt] = before + incl - len;
                s_b0[grp][gt] = start;
            }
            if (gt == 0) s_off[grp][n] = tot;
            group_sync(grp);  // also orders the table clear before the inserts
            chunk_products<kSG / 32>(s_off[grp], s_b0[grp], n, 0, tot, sc.heavy_pbuf,
                                     HashSink{table, kSSlots, &cnt, table_s});
        }
        cnt = static_cast<int>(warp_sum_ll(cnt));
        if (lane == 0 && cnt) {
            if (g.out)
                atomicAdd(reinterpret_cast<unsigned long long*>(&g.out[list[t.item]]),
                          static_cast<unsigned long long>(cnt));
            acc += cnt;
        }
        group_sync(grp);  // the table is free again
    }
    if (lane == 0 && acc)
        atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[g.total_slot]),
                  static_cast<unsigned long long>(acc));
}

// ======================================================= interval path
// B rows sorted (non-decreasing, the CsrMatrix invariant): the part of B row
// k inside a column interval is one contiguous run, so the columns are cut
// into P intervals of 2^shift <= 2^19 columns (interval_geometry) and a heavy
// row is counted interval by interval in a 64 KB shared bitmap, its products
// read straight from B -- no product buffer, no sort, no merge.  Per item and
// entry e the boundary table holds, for p = 1..P-1, the number of elements of
// e's B row below column p * 2^shift (row-relative).
//   bounds  per unit of products: 32 entries per warp step, one per lane;
//           slices longer than 32 elements are read by the whole warp
//           (coalesced) -- each element writes the boundaries it crosses;
//   plan    per item: exact product count of every interval (a pass over the
//           table), then tasks = runs of consecutive non-empty intervals with
//           at most kIntervalTarget products (one interval may exceed it);
//   run     two 512-thread blocks per SM take tasks off a counter; per
//           interval: clear the bitmap, stage the entries' runs (<= 2048 per
//           round), walk the products and count the bits set first.
struct IntervalTask {
    int32_t item;
    int32_t p0, p1;  // intervals [p0, p1)
    int32_t pad;
    int64_t products;
    int64_t pad2;
};
static_assert(sizeof(IntervalTask) == 32, "interval task layout");

constexpr int kIvBlock = 512;
constexpr int kIvItems = 4;                     // staged entries per thread
constexpr int kIvStage = kIvBlock * kIvItems;   // entries per staging round
constexpr int kIvSmem = (1 << kIvShift) / 8;    // the bitmap

__device__ __forceinline__ void set_bounds(int32_t* bnd, int64_t L, int64_t e, int from, int to, int32_t v) {
    for (int p = from; p <= to; ++p) bnd[static_cast<int64_t>(p - 1) * L + e] = v;
}

__global__ void __launch_bounds__(kHB) k_heavy_bounds(SymArgs g, SymScratch sc) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Intervals iv = interval_geometry(g.bcols);
    const int ks = iv.shift, P = iv.count;
    const long long units = sc.heavy_meta[0];
    // one warp per unit
    for (long long u = (blockIdx.x * int64_t(kHW) + w); u < units; u += int64_t(gridDim.x) * kHW) {
        const Unit un = find_unit(sc, 0, u);
        const int64_t i = un.item;
        const int64_t L = sc.heavy_eoff[i + 1] - sc.heavy_eoff[i] - 1;
        const int64_t* ep = sc.heavy_epre + sc.heavy_eoff[i];
        const int64_t* eb = sc.heavy_eb0 + sc.heavy_eoff[i];
        int32_t* bnd = sc.heavy_bnd + sc.heavy_boff[i];
        for (int64_t base = un.e0;; base += 32) {
            const int64_t e = base + lane;
            int64_t pe = 0, pn = 0, sb = 0, te = 0, b0 = 0;
            const bool in = e < L && (pe = ep[e]) < un.p1;
            if (in) {
                pn = ep[e + 1];
                sb = un.p0 > pe ? un.p0 - pe : 0;
                te = (pn < un.p1 ? pn : un.p1) - pe;
                b0 = eb[e];
            }
            if (!__any_sync(kFull, in)) break;  // past the unit's window
            const bool live = in && sb < te;
            const bool longs = live && te - sb > 32;
            if (live && !longs) {
                const int32_t* row = g.bcol + b0;
                int q[32];
                const int n = static_cast<int>(te - sb);
#pragma unroll
                for (int k = 0; k < 32; ++k) q[k] = k < n ? (__ldg(&row[sb + k]) >> ks) : 0;
                int prev = sb > 0 ? (__ldg(&row[sb - 1]) >> ks) : q[0];
#pragma unroll
                for (int k = 0; k < 32; ++k)
                    if (k < n) {
                        set_bounds(bnd, L, e, prev + 1, q[k] < P - 1 ? q[k] : P - 1, static_cast<int32_t>(sb + k));
                        prev = q[k];
                    }
                if (te == pn - pe) set_bounds(bnd, L, e, prev + 1, P - 1, static_cast<int32_t>(pn - pe));
            }
            for (unsigned m = __ballot_sync(kFull, longs); m; m &= m - 1) {
                const int src = __ffs(m) - 1;
                const int64_t ew = base + src;
                const int64_t s0 = __shfl_sync(kFull, sb, src), t0 = __shfl_sync(kFull, te, src);
                const int64_t len = __shfl_sync(kFull, pn - pe, src);
                const int32_t* row = g.bcol + __shfl_sync(kFull, b0, src);
                int qlast = 0;
                for (int64_t c = s0; c < t0; c += 32 * 4) {
                    int q[4], pv[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int64_t j = c + 32 * k + lane;
                        q[k] = j < t0 ? (__ldg(&row[j]) >> ks) : 0;
                        // the element before j (row start: no boundaries below it)
                        pv[k] = (lane == 0 && j < t0) ? (j > 0 ? (__ldg(&row[j - 1]) >> ks) : q[k]) : 0;
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int64_t j = c + 32 * k + lane;
                        int prev = __shfl_up_sync(kFull, q[k], 1);
                        if (lane == 0) prev = pv[k];
                        if (j < t0) set_bounds(bnd, L, ew, prev + 1, q[k] < P - 1 ? q[k] : P - 1, static_cast<int32_t>(j));
                        const int64_t left = t0 - (c + 32 * k);
                        if (left > 0) qlast = __shfl_sync(kFull, q[k], left < 32 ? static_cast<int>(left - 1) : 31);
                    }
                }
                if (t0 == len)
                    for (int p = qlast + 1 + lane; p <= P - 1; p += 32)
                        bnd[static_cast<int64_t>(p - 1) * L + ew] = static_cast<int32_t>(len);
            }
        }
    }
}

// One block per item: product count of every interval, then the tasks.
__global__ void __launch_bounds__(kHB) k_heavy_iplan(SymArgs g, SymScratch sc) {
    __shared__ long long s_cnt[kMaxIntervals];
    __shared__ int32_t s_t0[kMaxIntervals], s_t1[kMaxIntervals];
    __shared__ long long s_tp[kMaxIntervals];
    __shared__ int s_nt;
    __shared__ long long s_base;
    const int64_t i = blockIdx.x;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Intervals iv = interval_geometry(g.bcols);
    const int P = iv.count;
    const int64_t L = sc.heavy_eoff[i + 1] - sc.heavy_eoff[i] - 1;
    const int64_t* ep = sc.heavy_epre + sc.heavy_eoff[i];
    const int32_t* bnd = sc.heavy_bnd + sc.heavy_boff[i];
    for (int p = w; p < P; p += kHW) {
        long long c = 0;
        for (int64_t e = lane; e < L; e += 32) {
            const long long lo = p == 0 ? 0 : bnd[static_cast<int64_t>(p - 1) * L + e];
            const long long hi = p == P - 1 ? ep[e + 1] - ep[e] : bnd[static_cast<int64_t>(p) * L + e];
            c += hi - lo;
        }
        c = warp_sum_ll(c);
        if (lane == 0) s_cnt[p] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int nt = 0;
        long long acc = 0;
        for (int p = 0; p < P; ++p) {
            const long long c = s_cnt[p];
            if (c == 0) {  // an empty interval ends the run
                acc = 0;
                continue;
            }
            if (acc == 0 || acc + c > kIntervalTarget) {
                s_t0[nt] = p;
                s_tp[nt] = 0;
                ++nt;
                acc = 0;
            }
            acc += c;
            s_t1[nt - 1] = p + 1;
            s_tp[nt - 1] += c;
        }
        s_nt = nt;
        s_base = static_cast<long long>(atomicAdd(reinterpret_cast<unsigned long long*>(&sc.heavy_meta[3]),
                                                  static_cast<unsigned long long>(nt)));
    }
    __syncthreads();
    IntervalTask* out = reinterpret_cast<IntervalTask*>(sc.heavy_tasks) + s_base;
    for (int k = threadIdx.x; k < s_nt; k += kHB)
        out[k] = IntervalTask{static_cast<int32_t>(i), s_t0[k], s_t1[k], 0, s_tp[k], 0};
}

__global__ void __launch_bounds__(kIvBlock, 2) k_heavy_intervals(SymArgs g, SymScratch sc, int64_t first) {
    extern __shared__ int4 s_dyn_iv[];
    uint32_t* s_set = reinterpret_cast<uint32_t*>(s_dyn_iv);
    using Scan = cub::BlockScan<long long, kIvBlock>;
    __shared__ typename Scan::TempStorage s_scan;
    __shared__ int s_off[kIvStage + 1];
    __shared__ int64_t s_b0[kIvStage];
    __shared__ IntervalTask s_task;
    const IntervalTask* tasks = reinterpret_cast<const IntervalTask*>(sc.heavy_tasks);
    const int32_t* list = heavy_list(sc, first);
    const Intervals iv = interval_geometry(g.bcols);
    const int ks = iv.shift, P = iv.count;
    const int lane = threadIdx.x & 31;
    long long acc = 0;
    for (;;) {
        __syncthreads();  // the previous task is finished with the shared state
        if (threadIdx.x == 0) {
            const long long t = static_cast<long long>(
                atomicAdd(reinterpret_cast<unsigned long long*>(&sc.heavy_meta[7]), 1ULL));
            s_task = t < sc.heavy_meta[3] ? tasks[t] : IntervalTask{-1, 0, 0, 0, 0, 0};
        }
        __syncthreads();
        const IntervalTask t = s_task;
        if (t.item < 0) break;
        const int64_t i = t.item;
        const int64_t L = sc.heavy_eoff[i + 1] - sc.heavy_eoff[i] - 1;
        const int64_t* ep = sc.heavy_epre + sc.heavy_eoff[i];
        const int64_t* eb = sc.heavy_eb0 + sc.heavy_eoff[i];
        const int32_t* bnd = sc.heavy_bnd + sc.heavy_boff[i];
        int cnt = 0;
        for (int p = t.p0; p < t.p1; ++p) {
            const int c0 = p << ks;
            const int64_t width = (int64_t(p) + 1 << ks) < g.bcols ? (int64_t(1) << ks) : g.bcols - (int64_t(p) << ks);
            const int words = static_cast<int>((width + 31) >> 5);
            __syncthreads();  // the previous interval's inserts are done
            uint4* s4 = reinterpret_cast<uint4*>(s_set);
            for (int k = threadIdx.x; k < (words >> 2); k += kIvBlock) s4[k] = make_uint4(0u, 0u, 0u, 0u);
            for (int k = (words & ~3) + threadIdx.x; k < words; k += kIvBlock) s_set[k] = 0u;
            for (int64_t e0 = 0; e0 < L; e0 += kIvStage) {
                const int n = static_cast<int>(L - e0 < kIvStage ? L - e0 : kIvStage);
                long long len[kIvItems];
                int64_t start[kIvItems];
#pragma unroll
                for (int k = 0; k < kIvItems; ++k) {
                    const int j = threadIdx.x * kIvItems + k;
                    len[k] = 0;
                    start[k] = 0;
                    if (j < n) {
                        const int64_t e = e0 + j;
                        const int64_t lo = p == 0 ? 0 : bnd[static_cast<int64_t>(p - 1) * L + e];
                        const int64_t hi = p == P - 1 ? ep[e + 1] - ep[e] : bnd[static_cast<int64_t>(p) * L + e];
                        len[k] = hi - lo;
                        start[k] = eb[e] + lo;
                    }
                }
                long long ex[kIvItems], tot;
                __syncthreads();  // the clear is done / the previous round's walk is done
                Scan(s_scan).ExclusiveSum(len, ex, tot);
#pragma unroll
                for (int k = 0; k < kIvItems; ++k) {
                    const int j = threadIdx.x * kIvItems + k;
                    if (j < n) {
                        s_off[j] = static_cast<int>(ex[k]);
                        s_b0[j] = start[k];
                    }
                }
                if (threadIdx.x == 0) s_off[n] = static_cast<int>(tot);
                __syncthreads();
                chunk_products<kIvBlock / 32>(s_off, s_b0, n, 0, static_cast<int>(tot), g.bcol,
                                              [&](const int (&keys)[kUnroll], const bool (&valid)[kUnroll], long long) {
#pragma unroll
                                                  for (int v = 0; v < kUnroll; ++v)
                                                      if (valid[v]) {
                                                          const uint32_t off = static_cast<uint32_t>(keys[v] - c0);
                                                          SPNNZ_ASSERT((off >> 5) < static_cast<uint32_t>(kIvSmem / 4));
                                                          const uint32_t bit = 1u << (off & 31);
                                                          cnt += (atomicOr(&s_set[off >> 5], bit) & bit) ? 0 : 1;
                                                      }
                                              });
            }
        }
        cnt = static_cast<int>(warp_sum_ll(cnt));
        if (lane == 0 && cnt) {
            if (g.out)
                atomicAdd(reinterpret_cast<unsigned long long*>(&g.out[list[i]]),
                          static_cast<unsigned long long>(cnt));
            acc += cnt;
        }
    }
    if (lane == 0 && acc)
        atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[g.total_slot]),
                  static_cast<unsigned long long>(acc));
}

// FLOP, A-row length and boundary cells of every heavy item (host batch
// planning in exact mode).
__global__ void k_heavy_flops(SymArgs g, SymScratch sc, int64_t count, int64_t* out) {
    const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (i >= count) return;
    const int32_t s = heavy_list(sc, 0)[i];
    const int32_t rid = g.rows ? g.rows[s] : g.row_lo + s;
    const int32_t r = rid - g.row_lo;
    const int64_t L = g.a.rpt[r + 1] - g.a.rpt[r];
    out[i] = g.item_flop ? g.item_flop[s] : g.flop[r];
    out[count + i] = L;
    out[2 * count + i] = (interval_geometry(g.bcols).count - 1) * L;
}

int sort_smem(int R) { return int(2 * kHeavyUnitProducts * 4 + ((kHW + 1) * R + 1) * 4); }

int place_smem() { return int(kMaxRanges * 8 + 2 * kHeavyUnitProducts * 4 + kMaxRanges * 4 + (kMaxRanges + 1) * 4); }

}  // namespace

HeavyGeometry heavy_geometry(int32_t bcols) {
    HeavyGeometry h;
    int lg = 5;
    while ((int64_t(1) << lg) < bcols) ++lg;  // 2^lg >= B.cols
    if (lg <= kSpanShift) {
        h.wshift = lg;
        h.ranges = 1;
    } else {
        const int ws = kTaskSpanShift;  // one range per task span
        h.wshift = ws;
        h.ranges = static_cast<int>((int64_t(bcols) + (int64_t(1) << ws) - 1) >> ws);
        h.unit_sorted = h.ranges <= kPrivRanges;
    }
    // words of a merge slot: a task span (R > 1) or the whole row (R == 1)
    h.wwords = h.ranges > 1 ? (1 << kTaskSpanShift) / 32
                            : static_cast<int32_t>(((int64_t(1) << h.wshift) + 31) / 32);
    return h;
}

int64_t heavy_task_bound(int64_t count, int64_t products, int ranges) {
    // one task per span of every item, plus the extra parts of split spans
    return count * (int64_t(ranges) + 1) + 2 * (products / kTaskProducts + 1);
}

int64_t heavy_slot_bound(int64_t, int64_t products) {
    // a merge slot serves one span (or row) that needs >= 2 tasks
    return products / kTaskProducts + 1;
}

cudaError_t launch_heavy_flops(const SymArgs& args, const SymScratch& s, int64_t count,
                               int64_t* out, cudaStream_t stream) {
    if (count == 0) return cudaSuccess;
    k_heavy_flops<<<static_cast<unsigned>((count + 255) / 256), 256, 0, stream>>>(args, s, count, out);
    return cudaGetLastError();
}

// debug timeline (SPNNZ_DEBUG_TIMELINE): events after each heavy kernel
static cudaEvent_t g_hev[12] = {};
static const char* g_hname[12] = {};
static int g_hn = 0;
static bool g_hdbg = false;
static void hmark(const char* name, cudaStream_t st) {
    if (!g_hdbg || g_hn >= 12) return;
    if (!g_hev[g_hn]) cudaEventCreate(&g_hev[g_hn]);
    g_hname[g_hn] = name;
    cudaEventRecord(g_hev[g_hn++], st);
}
void heavy_debug_print(cudaEvent_t start) {
    for (int i = 0; i < g_hn; ++i) {
        float t = 0.f;
        cudaEventElapsedTime(&t, start, g_hev[i]);
        fprintf(stderr, "  heavy %s end %.1f us\n", g_hname[i], 1e3 * t);
    }
    g_hn = 0;
}

cudaError_t launch_sym_heavy(const SymArgs& args, const SymScratch& s, bool sorted, int64_t first,
                             int64_t count, int num_sms, cudaStream_t stream, int64_t* launches,
                             cudaStream_t aux, cudaEvent_t ev_a, cudaEvent_t ev_b, cudaEvent_t run_gate) {
    if (count == 0) return cudaSuccess;
    int64_t n = 0;  // kernels launched (memsets not counted)
    static std::atomic<unsigned long long> attr_done{0};  // one bit per device; the sets are idempotent
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_done.load(std::memory_order_acquire) & (1ull << (dev & 63)))) {
        cudaFuncSetAttribute(k_heavy_run<1024, kRunItem>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (1 << kSpanShift) / 8);
        cudaFuncSetAttribute(k_heavy_run<1024, kRunItem, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (1 << kSpanShift) / 8);
        cudaFuncSetAttribute(k_heavy_run<512, kRunBuckets>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (1 << kTaskSpanShift) / 8);
        cudaFuncSetAttribute(k_heavy_run_units<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (1 << kTaskSpanShift) / 8);
        cudaFuncSetAttribute(k_heavy_run_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSGroups * kSSlots * 4);
        cudaFuncSetAttribute(k_heavy_place, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             place_smem());
        cudaFuncSetAttribute(k_heavy_sort_units, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             sort_smem(kPrivRanges));
        cudaFuncSetAttribute(k_heavy_intervals, cudaFuncAttributeMaxDynamicSharedMemorySize, kIvSmem);
        attr_done.fetch_or(1ull << (dev & 63), std::memory_order_release);
    }
    const HeavyGeometry geo = heavy_geometry(args.bcols);
    const int R = geo.ranges;
    const unsigned sms = static_cast<unsigned>(num_sms);
    const unsigned items = static_cast<unsigned>(count);
    g_hdbg = getenv("SPNNZ_DEBUG_TIMELINE") != nullptr;
    g_hn = 0;
    k_heavy_prep<<<1, kPrepBlock, 0, stream>>>(args, s, first, count);
    hmark("prep", stream);
    k_heavy_entries<<<items, kEntB, 0, stream>>>(args, s, first);
    hmark("entries", stream);
    n += 2;
    if (sorted) {
        cudaMemsetAsync(s.heavy_bnd, 0, sizeof(int32_t) * s.heavy_bnd_cap, stream);
        k_heavy_bounds<<<sms * 8, kHB, 0, stream>>>(args, s);
        k_heavy_iplan<<<items, kHB, 0, stream>>>(args, s);
        k_heavy_intervals<<<sms * 2, kIvBlock, kIvSmem, stream>>>(args, s, first);
        if (launches) *launches += n + 3;
        return cudaGetLastError();
    }
    if (R > 1) {
        cudaMemsetAsync(s.heavy_rc, 0, sizeof(long long) * count * R, stream);
        if (geo.unit_sorted) {
            k_heavy_sort_units<<<sms * (1536 / kHB), kHB, sort_smem(R), stream>>>(args, s, first, count, R, geo.wshift);
            hmark("sort", stream);
            k_heavy_plan_units<<<items, kPrivRanges, 0, stream>>>(s, count, R, s.heavy_task_cap);
            hmark("plan", stream);
            if (run_gate) cudaStreamWaitEvent(stream, run_gate, 0);  // the runs after the gate (FLOP pass)
            // the bitmap tasks and the small hash tasks are independent: on
            // two streams (aux given) each fills the other's tail
            if (aux) {
                cudaEventRecord(ev_a, stream);
                cudaStreamWaitEvent(aux, ev_a, 0);
            }
            k_heavy_run_units<512><<<sms * SPNNZ_RUN_GRID, 512, (1 << kTaskSpanShift) / 8, stream>>>(
                args, s, first, R, geo.wshift, geo.wwords);
            hmark("run_units", stream);
            k_heavy_run_small<<<sms * 3, kSG * kSGroups, kSGroups * kSSlots * 4, aux ? aux : stream>>>(
                args, s, first, R);
            hmark("run_small", aux ? aux : stream);
            if (aux) {
                cudaEventRecord(ev_b, aux);
                cudaStreamWaitEvent(stream, ev_b, 0);
            }
            n += 4;
        } else {
            k_heavy_count<<<sms * 8, kHB, 0, stream>>>(args, s, first, count, R, geo.wshift);
            k_heavy_offsets<<<items, 256, 0, stream>>>(s, count, R);
            k_heavy_place<<<sms * 2, kHB, place_smem(), stream>>>(args, s, first,
                                                                             count, R, geo.wshift);
            k_heavy_plan<<<items, 128, 0, stream>>>(s, count, R, geo.wshift, s.heavy_task_cap);
            n += 5;
            k_heavy_run<512, kRunBuckets><<<sms * 3, 512, (1 << kTaskSpanShift) / 8, stream>>>(
                args, s, first, R, geo.wshift, geo.wwords);
        }
    } else {
        k_heavy_tasks_r1<<<static_cast<unsigned>((count + 127) / 128), 128, 0, stream>>>(
            s, count, s.heavy_task_cap);
        // swizzled bitmap layout (bank = the column's low five bits) for spans
        // of >= 2^10 bits; A/B knob SPNNZ_BITMAP_SWZ=0
        static const bool swz_on = [] {
            const char* e = getenv("SPNNZ_BITMAP_SWZ");
            return !(e && atoi(e) == 0);
        }();
        if (swz_on && geo.wshift >= 10)
            k_heavy_run<1024, kRunItem, true><<<sms, 1024, (1 << kSpanShift) / 8, stream>>>(
                args, s, first, R, geo.wshift, geo.wwords);
        else
            k_heavy_run<1024, kRunItem><<<sms, 1024, (1 << kSpanShift) / 8, stream>>>(
                args, s, first, R, geo.wshift, geo.wwords);
        n += 2;
    }
    k_heavy_slot_count<<<sms * 4, kSlotBlock, 0, stream>>>(args, s, first, int64_t(geo.wwords));
    if (launches) *launches += n + 1;
    return cudaGetLastError();
}

}  // namespace spnnz_gpu
