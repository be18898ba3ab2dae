// Heavy rows of the symbolic engine (FLOP > kBin5Max): exact distinct-column
// counts with every set operation in shared memory.
//
// A heavy row of C = A*B can have millions of products (config 5: 8.5 M) and
// its distinct set does not fit one SM.  A per-row global bitmap (2 MB at
// config 5, ~850 rows in flight) thrashes L2 into gigabytes of DRAM
// read-modify-write, so instead the row's products are bucketed by column
// range and every bucket is counted on chip in a shared-memory bitmap:
//   0. prep/entries  per batch: unit, entry and product offsets of every
//                    heavy row; per row, the product prefix over its entries;
//   1. count    per unit of kHeavyUnitProducts products (one block): per-warp
//               shared histograms over the R column ranges of width W;
//   2. offsets  per row, bucket starts in the product buffer;
//   3. scatter  per unit again: stage the products in shared memory, count
//               them per warp and range, reserve each range's slice with one
//               global atomic, and write them out grouped by range;
//   4. tasks    per row, consecutive ranges are packed into tasks spanning at
//               most 2^20 columns (a 128 KB shared bitmap) and at most
//               kTaskProducts products; a range with more products is split
//               into several tasks that share a merge slot;
//   5. run      one 1024-thread block per task: clear the span's bitmap,
//               atomicOr each product's bit and count the bits it set first.
//               Tasks that share a range then OR their non-zero words into a
//               global W-bit merge bitmap and count popc(word & ~old) instead.
// B.cols <= 2^20 (configs 2 and 4): one range covers all columns, steps 1-3
// are skipped and tasks read their product slice straight from the B rows.
// W = max(2^17, 2^ceil(log2 B.cols) / 256) keeps R <= 256 (per-warp
// histograms) up to B.cols = 2^28; beyond that W = 2^20 and the histograms
// are shared.  Every count is a set cardinality: exact and independent of
// bucketing, task boundaries and scheduling.
#include "symbolic_common.cuh"

namespace spnnz_gpu {
namespace {
using namespace sym;

constexpr int kHB = 256;                  // block of the unit passes
constexpr int kHW = kHB / 32;             // warps per unit block
constexpr int kRunBlock = 1024;           // block of the task runner
constexpr int kSpanShift = 20;            // task column span <= 2^20 (128 KB)
constexpr int kPrivRanges = 256;          // per-warp histograms up to this R
constexpr int kMaxRanges = 2048;          // B.cols < 2^31 with W = 2^20
constexpr int64_t kTaskProducts = 131072;

struct HeavyTask {
    int32_t item;      // index in the batch
    int32_t slot;      // merge bitmap slot, or -1
    int32_t col_base;  // first column of the task's span
    int32_t words;     // span / 32 (bitmap words to clear)
    int64_t p0, p1;    // R > 1: product-buffer span; R == 1: the item's product range
};
static_assert(sizeof(HeavyTask) == 32, "task layout");

__device__ __forceinline__ const int32_t* heavy_list(const SymScratch& sc, int64_t first) {
    return sc.lists + int64_t(kHeavyBin) * sc.capacity + first;
}

// ---- 0a. batch bookkeeping: units, entry offsets, product offsets (1 block)
__global__ void __launch_bounds__(256) k_heavy_prep(SymArgs g, SymScratch sc, int64_t first,
                                                    int64_t count) {
    using Scan = cub::BlockScan<long long, 256>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ long long s_u, s_e, s_f;
    if (threadIdx.x == 0) s_u = s_e = s_f = 0;
    __syncthreads();
    const int32_t* list = heavy_list(sc, first);
    for (int64_t b = 0; b < count; b += 256) {
        const int64_t i = b + threadIdx.x;
        long long units = 0, ents = 0, f = 0;
        if (i < count) {
            const int32_t s = list[i];
            const int32_t rid = g.rows ? g.rows[s] : g.row_lo + s;
            const ItemRow it = item_row(g, s);
            f = g.flop[rid - g.row_lo];
            units = (f + kHeavyUnitProducts - 1) / kHeavyUnitProducts;
            ents = it.a1 - it.a0 + 1;
        }
        long long ue, ee, fe, ut, et, ft;
        Scan(tmp).ExclusiveSum(units, ue, ut);
        __syncthreads();
        Scan(tmp).ExclusiveSum(ents, ee, et);
        __syncthreads();
        Scan(tmp).ExclusiveSum(f, fe, ft);
        if (i < count) {
            sc.heavy_unit_off[i] = s_u + ue;
            sc.heavy_eoff[i] = s_e + ee;
            sc.heavy_foff[i] = s_f + fe;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s_u += ut;
            s_e += et;
            s_f += ft;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        sc.heavy_unit_off[count] = s_u;
        sc.heavy_eoff[count] = s_e;
        sc.heavy_foff[count] = s_f;
        sc.heavy_meta[0] = s_u;
        sc.heavy_meta[3] = 0;  // tasks
        sc.heavy_meta[4] = 0;  // merge slots
    }
}

// ---- 0b. one block per item: product prefix over its entries, B-row starts
__global__ void __launch_bounds__(256) k_heavy_entries(SymArgs g, SymScratch sc, int64_t first) {
    using Scan = cub::BlockScan<long long, 256>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ long long s_carry;
    const int64_t i = blockIdx.x;
    const ItemRow it = item_row(g, heavy_list(sc, first)[i]);
    int64_t* ep = sc.heavy_epre + sc.heavy_eoff[i];
    int64_t* eb = sc.heavy_eb0 + sc.heavy_eoff[i];
    const int64_t L = it.a1 - it.a0;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < L; c0 += 256) {
        const int64_t e = c0 + threadIdx.x;
        long long d = 0;
        int64_t b0 = 0;
        if (e < L) {
            const int c = __ldg(&g.a.col[it.a0 + e]);
            b0 = __ldg(&g.brpt[c]);
            d = __ldg(&g.brpt[c + 1]) - b0;
        }
        long long ex, tot;
        Scan(tmp).ExclusiveSum(d, ex, tot);
        if (e < L) {
            ep[e] = s_carry + ex;
            eb[e] = b0;
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
};

__device__ __forceinline__ Unit find_unit(const SymScratch& sc, int64_t count, long long u) {
    int64_t lo = 0, hi = count - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (sc.heavy_unit_off[mid] <= u) lo = mid; else hi = mid - 1;
    }
    Unit r;
    r.item = lo;
    const long long ftot = sc.heavy_foff[lo + 1] - sc.heavy_foff[lo];
    r.p0 = (u - sc.heavy_unit_off[lo]) * kHeavyUnitProducts;
    r.p1 = r.p0 + kHeavyUnitProducts < ftot ? r.p0 + kHeavyUnitProducts : ftot;
    return r;
}

// Block-wide walk over products [p0, p1) of heavy item `item` (p1 - p0 <
// 2^31): chunks of BLOCK entries are staged in shared memory with offsets
// relative to p0 (clamped to [0, p1 - p0], B-row starts shifted to match) so
// the per-product cursor works in 32-bit.  fn(keys, valid, q) with keys[u]
// = product p0 + q + 32 u.
template <int BLOCK, typename Fn>
__device__ __forceinline__ void item_products(const SymArgs& g, const SymScratch& sc,
                                              int64_t first, int64_t item, long long p0,
                                              long long p1, int* s_off, int64_t* s_b0, Fn&& fn) {
    const ItemRow it = item_row(g, heavy_list(sc, first)[item]);
    const int64_t L = it.a1 - it.a0;
    const int64_t* ep = sc.heavy_epre + sc.heavy_eoff[item];
    const int64_t* eb = sc.heavy_eb0 + sc.heavy_eoff[item];
    const long long span = p1 - p0;
    int64_t e0 = 0, e1 = L - 1;  // largest entry with ep[e] <= p0
    while (e0 < e1) {
        const int64_t mid = (e0 + e1 + 1) >> 1;
        if (ep[mid] <= p0) e0 = mid; else e1 = mid - 1;
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
        chunk_products<BLOCK / 32>(s_off, s_b0, n, s_off[0], s_off[n], g.bcol, fn);
        const bool done = s_off[n] >= span || e + n >= L;
        if (done) break;
        e += n;
    }
    __syncthreads();
}

// ---- 1. per-unit histogram over column ranges
template <bool PRIV>
__global__ void __launch_bounds__(kHB) k_heavy_count(SymArgs g, SymScratch sc, int64_t first,
                                                     int64_t count, int R, int wshift) {
    constexpr int NW = PRIV ? kHW : 1, RM = PRIV ? kPrivRanges : kMaxRanges;
    __shared__ int s_off[kHB + 1];
    __shared__ int64_t s_b0[kHB];
    __shared__ int s_hist[NW][RM];
    const int w = PRIV ? threadIdx.x >> 5 : 0;
    const long long units = sc.heavy_meta[0];
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        const Unit un = find_unit(sc, count, u);
        for (int k = threadIdx.x; k < NW * R; k += kHB) s_hist[k / R][k % R] = 0;
        item_products<kHB>(g, sc, first, un.item, un.p0, un.p1, s_off, s_b0,
                           [&](const int (&keys)[kUnroll], const bool (&valid)[kUnroll], long long) {
#pragma unroll
                               for (int k = 0; k < kUnroll; ++k)
                                   if (valid[k]) atomicAdd(&s_hist[w][keys[k] >> wshift], 1);
                           });
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

// ---- 2. bucket offsets (exclusive prefix per item, placed at foff[item])
__global__ void k_heavy_offsets(SymScratch sc, int64_t count, int R) {
    const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (i >= count) return;
    long long acc = sc.heavy_foff[i];
    long long* rc = sc.heavy_rc + i * R;
    long long* cur = sc.heavy_cur + i * R;
    for (int r = 0; r < R; ++r) {
        const long long c = rc[r];
        rc[r] = acc;
        cur[r] = acc;
        acc += c;
    }
}

// ---- 3. scatter products into their range buckets
template <bool PRIV>
__global__ void __launch_bounds__(kHB) k_heavy_scatter(SymArgs g, SymScratch sc, int64_t first,
                                                       int64_t count, int R, int wshift) {
    constexpr int NW = PRIV ? kHW : 1, RM = PRIV ? kPrivRanges : kMaxRanges;
    __shared__ int s_off[kHB + 1];
    __shared__ int64_t s_b0[kHB];
    __shared__ int s_hist[NW][RM];      // counts, then per-warp cursors
    __shared__ long long s_base[RM];    // global start of the unit's slice per range
    extern __shared__ int4 s_dyn_keys[];
    int32_t* s_keys = reinterpret_cast<int32_t*>(s_dyn_keys);  // kHeavyUnitProducts
    const int w = PRIV ? threadIdx.x >> 5 : 0;
    const long long units = sc.heavy_meta[0];
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        const Unit un = find_unit(sc, count, u);
        for (int k = threadIdx.x; k < NW * R; k += kHB) s_hist[k / R][k % R] = 0;
        item_products<kHB>(g, sc, first, un.item, un.p0, un.p1, s_off, s_b0,
                           [&](const int (&keys)[kUnroll], const bool (&valid)[kUnroll],
                               long long q) {
#pragma unroll
                               for (int k = 0; k < kUnroll; ++k)
                                   if (valid[k]) s_keys[q + 32 * k] = keys[k];
                           });
        const int n = static_cast<int>(un.p1 - un.p0);
        for (int i = threadIdx.x; i < n; i += kHB) atomicAdd(&s_hist[w][s_keys[i] >> wshift], 1);
        __syncthreads();
        // per range: reserve the unit's slice, turn the counts into per-warp offsets
        long long* cur = sc.heavy_cur + un.item * R;
        for (int r = threadIdx.x; r < R; r += kHB) {
            int tot = 0;
#pragma unroll
            for (int v = 0; v < NW; ++v) {
                const int c = s_hist[v][r];
                s_hist[v][r] = tot;
                tot += c;
            }
            s_base[r] = tot ? static_cast<long long>(atomicAdd(
                                  reinterpret_cast<unsigned long long*>(&cur[r]),
                                  static_cast<unsigned long long>(tot)))
                            : 0;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += kHB) {  // same thread <-> item mapping
            const int key = s_keys[i];
            const int r = key >> wshift;
            sc.heavy_pbuf[s_base[r] + atomicAdd(&s_hist[w][r], 1)] = key;
        }
        __syncthreads();
    }
}

// ---- 4. tasks per item (one thread per item; appends with one atomic)
// Builds item i's task list; with out == nullptr it only counts.
__device__ int build_tasks(const SymScratch& sc, int64_t i, int R, int wshift, int32_t bcols,
                           HeavyTask* out) {
    const int32_t item = static_cast<int32_t>(i);
    int k = 0;
    // [p0, p1) products of one span starting at column `base`, `words` wide
    auto emit = [&](int32_t base, int32_t words, long long p0, long long p1) {
        const long long parts = (p1 - p0 + kTaskProducts - 1) / kTaskProducts;
        int32_t slot = -1;
        if (out && parts > 1)
            slot = static_cast<int32_t>(
                atomicAdd(reinterpret_cast<unsigned long long*>(&sc.heavy_meta[4]), 1ULL));
        for (long long q = 0; q < parts; ++q, ++k) {
            if (!out) continue;
            const long long a = p0 + q * kTaskProducts;
            const long long b = a + kTaskProducts < p1 ? a + kTaskProducts : p1;
            out[k] = HeavyTask{item, slot, base, words, a, b};
        }
    };
    if (R == 1) {  // whole row in one span, read from the B rows
        emit(0, static_cast<int32_t>((int64_t(bcols) + 31) / 32), 0,
             sc.heavy_foff[i + 1] - sc.heavy_foff[i]);
        return k;
    }
    const int per_span = 1 << (kSpanShift - wshift);  // ranges per 2^20-column span
    const int32_t wwords = static_cast<int32_t>((int64_t(1) << wshift) / 32);
    const long long* rc = sc.heavy_rc + i * R;
    const long long end = sc.heavy_foff[i + 1];
    int g0 = -1, g1 = -1;  // open group of ranges [g0, g1)
    auto flush = [&]() {
        if (g0 >= 0) {
            const long long a = rc[g0], b = g1 < R ? rc[g1] : end;
            if (b > a) {
                if (out) out[k] = HeavyTask{item, -1, g0 << wshift, (g1 - g0) * wwords, a, b};
                ++k;
            }
        }
        g0 = g1 = -1;
    };
    for (int r = 0; r < R; ++r) {
        const long long b0 = rc[r];
        const long long b1 = r + 1 < R ? rc[r + 1] : end;
        if (b1 == b0) continue;
        if (b1 - b0 > kTaskProducts) {  // one range, several tasks, merged
            flush();
            emit(r << wshift, wwords, b0, b1);
        } else if (g0 >= 0 && r + 1 - g0 <= per_span && b1 - rc[g0] <= kTaskProducts) {
            g1 = r + 1;
        } else {
            flush();
            g0 = r;
            g1 = r + 1;
        }
    }
    flush();
    return k;
}

__global__ void k_heavy_tasks(SymScratch sc, int64_t count, int R, int wshift, int32_t bcols,
                              int64_t task_cap) {
    const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (i >= count) return;
    const int n = build_tasks(sc, i, R, wshift, bcols, nullptr);
    const long long base = static_cast<long long>(atomicAdd(
        reinterpret_cast<unsigned long long*>(&sc.heavy_meta[3]), static_cast<unsigned long long>(n)));
    if (base + n > task_cap) __trap();  // host sizes task_cap to heavy_task_bound()
    build_tasks(sc, i, R, wshift, bcols, reinterpret_cast<HeavyTask*>(sc.heavy_tasks) + base);
}

// ---- 5. run the tasks: one block per task, a <= 2^20-bit shared bitmap
__global__ void __launch_bounds__(kRunBlock) k_heavy_run(SymArgs g, SymScratch sc, int64_t first,
                                                         int R, int wshift) {
    extern __shared__ int4 s_dyn[];
    uint32_t* s_set = reinterpret_cast<uint32_t*>(s_dyn);
    __shared__ int s_off[kRunBlock + 1];
    __shared__ int64_t s_b0[kRunBlock];
    __shared__ long long s_red[kRunBlock / 32];
    const HeavyTask* tasks = reinterpret_cast<const HeavyTask*>(sc.heavy_tasks);
    const long long ntask = sc.heavy_meta[3];
    const int32_t* list = heavy_list(sc, first);
    const int32_t wwords = static_cast<int32_t>((int64_t(1) << wshift) / 32);
    long long acc = 0;
    for (long long ti = blockIdx.x; ti < ntask; ti += gridDim.x) {
        const HeavyTask t = tasks[ti];
        for (int k = threadIdx.x; k < t.words; k += kRunBlock) s_set[k] = 0u;
        __syncthreads();
        int cnt = 0;
        auto insert = [&](const int (&keys)[kUnroll], const bool (&valid)[kUnroll], long long) {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
                if (valid[u]) {
                    const uint32_t off = static_cast<uint32_t>(keys[u] - t.col_base);
                    const uint32_t bit = 1u << (off & 31);
                    cnt += (atomicOr(&s_set[off >> 5], bit) & bit) ? 0 : 1;
                }
        };
        if (R > 1) {
            for (long long p = t.p0 + threadIdx.x; p < t.p1; p += kRunBlock * kUnroll) {
                int keys[kUnroll];
                bool valid[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const long long q = p + u * kRunBlock;
                    valid[u] = q < t.p1;
                    keys[u] = valid[u] ? __ldg(&sc.heavy_pbuf[q]) : 0;
                }
                insert(keys, valid, 0);
            }
        } else {
            item_products<kRunBlock>(g, sc, first, t.item, t.p0, t.p1, s_off, s_b0, insert);
        }
        if (t.slot >= 0) {
            // range shared by several tasks: the bits this task adds first
            __syncthreads();
            cnt = 0;
            uint32_t* gbm = sc.pool + int64_t(t.slot) * wwords;
            for (int k = threadIdx.x; k < t.words; k += kRunBlock) {
                const uint32_t w = s_set[k];
                if (w) cnt += __popc(w & ~atomicOr(&gbm[k], w));
            }
        }
        const long long tot = block_sum_ll<kRunBlock>(cnt, s_red);
        if (threadIdx.x == 0 && tot) {
            if (g.out)
                atomicAdd(reinterpret_cast<unsigned long long*>(&g.out[list[t.item]]),
                          static_cast<unsigned long long>(tot));
            acc += tot;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && acc)
        atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[g.total_slot]),
                  static_cast<unsigned long long>(acc));
}

// FLOP of every heavy item (for the host's batch planning in exact mode).
__global__ void k_heavy_flops(SymArgs g, SymScratch sc, int64_t count, int64_t* out) {
    const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (i >= count) return;
    const int32_t s = heavy_list(sc, 0)[i];
    const int32_t rid = g.rows ? g.rows[s] : g.row_lo + s;
    out[i] = g.flop[rid - g.row_lo];
}

// ---- 6. return the used merge bitmaps to zero
__global__ void k_heavy_clean(SymScratch sc, int64_t slot_words) {
    const long long used = sc.heavy_meta[4] * slot_words;
    for (long long i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < used;
         i += int64_t(gridDim.x) * blockDim.x)
        sc.pool[i] = 0u;
}

}  // namespace

HeavyGeometry heavy_geometry(int32_t bcols) {
    HeavyGeometry h;
    int lg = 5;
    while ((int64_t(1) << lg) < bcols) ++lg;  // 2^lg >= B.cols
    if (lg <= kSpanShift) {
        h.wshift = lg;
        h.ranges = 1;
    } else {
        int ws = lg - 8;  // R <= 256
        if (ws < 17) ws = 17;
        if (ws > kSpanShift) ws = kSpanShift;
        h.wshift = ws;
        h.ranges = static_cast<int>((int64_t(bcols) + (int64_t(1) << ws) - 1) >> ws);
    }
    h.wwords = static_cast<int32_t>(((int64_t(1) << h.wshift) + 31) / 32);
    return h;
}

int64_t heavy_task_bound(int64_t count, int64_t products, int ranges) {
    // groups: at most one per non-empty range, plus split parts
    return count * (int64_t(ranges) + 1) + 2 * (products / kTaskProducts + 1);
}

int64_t heavy_slot_bound(int64_t, int64_t products) {
    // a merge slot serves one range (or row) that needs >= 2 tasks
    return products / kTaskProducts + 1;
}

cudaError_t launch_heavy_flops(const SymArgs& args, const SymScratch& s, int64_t count,
                               int64_t* out, cudaStream_t stream) {
    if (count == 0) return cudaSuccess;
    k_heavy_flops<<<static_cast<unsigned>((count + 255) / 256), 256, 0, stream>>>(args, s, count, out);
    return cudaGetLastError();
}

cudaError_t launch_sym_heavy(const SymArgs& args, const SymScratch& s, int64_t first,
                             int64_t count, int num_sms, cudaStream_t stream) {
    if (count == 0) return cudaSuccess;
    static unsigned attr_done = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_done & (1u << (dev & 31)))) {
        cudaFuncSetAttribute(k_heavy_run, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (1 << kSpanShift) / 8);
        cudaFuncSetAttribute(k_heavy_scatter<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(kHeavyUnitProducts * 4));
        cudaFuncSetAttribute(k_heavy_scatter<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(kHeavyUnitProducts * 4));
        attr_done |= 1u << (dev & 31);
    }
    const HeavyGeometry geo = heavy_geometry(args.bcols);
    const int R = geo.ranges;
    k_heavy_prep<<<1, 256, 0, stream>>>(args, s, first, count);
    k_heavy_entries<<<static_cast<unsigned>(count), 256, 0, stream>>>(args, s, first);
    const unsigned sms = static_cast<unsigned>(num_sms);
    if (R > 1) {
        cudaMemsetAsync(s.heavy_rc, 0, sizeof(long long) * count * R, stream);
        const int keys_smem = int(kHeavyUnitProducts * 4);
        if (R <= kPrivRanges) {
            k_heavy_count<true><<<sms * 8, kHB, 0, stream>>>(args, s, first, count, R, geo.wshift);
            k_heavy_offsets<<<static_cast<unsigned>((count + 255) / 256), 256, 0, stream>>>(s, count, R);
            k_heavy_scatter<true><<<sms * 4, kHB, keys_smem, stream>>>(args, s, first, count, R,
                                                                       geo.wshift);
        } else {
            k_heavy_count<false><<<sms * 8, kHB, 0, stream>>>(args, s, first, count, R, geo.wshift);
            k_heavy_offsets<<<static_cast<unsigned>((count + 255) / 256), 256, 0, stream>>>(s, count, R);
            k_heavy_scatter<false><<<sms * 2, kHB, keys_smem, stream>>>(args, s, first, count, R,
                                                                        geo.wshift);
        }
    }
    k_heavy_tasks<<<static_cast<unsigned>((count + 127) / 128), 128, 0, stream>>>(
        s, count, R, geo.wshift, args.bcols, s.heavy_task_cap);
    k_heavy_run<<<sms, kRunBlock, (1 << kSpanShift) / 8, stream>>>(args, s, first, R, geo.wshift);
    k_heavy_clean<<<sms * 4, 256, 0, stream>>>(s, int64_t(geo.wwords));
    return cudaGetLastError();
}

}  // namespace spnnz_gpu
