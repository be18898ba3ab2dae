// Heavy rows of the symbolic engine (FLOP > kBin5Max): exact distinct-column
// counts with every set operation in shared memory.
//
// A heavy row of C = A*B can have millions of products (config 5: 8.5 M) and
// its distinct set does not fit one SM.  Instead of a per-row global bitmap
// (B.cols bits: 2 MB at config 5, ~1000 rows in flight => gigabytes of
// random read-modify-write traffic that thrashes L2), the row's products are
// bucketed by column range and every bucket is counted on chip:
//   1. count    per unit of kHeavyUnitProducts products (one block), a
//               shared histogram over the R column ranges of width W
//               (W = min(B.cols, 2^20) bits, R = ceil(B.cols / W));
//   2. offsets  per row, bucket starts in a product buffer (prefix of the
//               histogram, per-row spans laid out by an item prefix of FLOP);
//   3. scatter  per unit again: stage the unit's products in shared memory,
//               reserve each range's slice with one global atomic, and write
//               the products out grouped by range;
//   4. tasks    per row, consecutive ranges are packed into tasks of at most
//               kHashTaskProducts products (shared hash of 49152 slots); a
//               range with more products becomes bitmap tasks of at most
//               kBitmapTaskProducts products each (shared bitmap of W bits);
//   5. run      one block per task; a bitmap task that shares its range with
//               other tasks ORs its non-zero words into a global W-bit merge
//               bitmap and counts popc(word & ~old): the bits it added first.
// When R == 1 (B.cols <= 2^20: configs 2 and 4) steps 1-3 are skipped and
// bitmap tasks enumerate their product range straight from the B rows.
// Every count is a set cardinality, so the result is exact and independent
// of bucketing, task boundaries and scheduling.
#include "symbolic_common.cuh"

namespace spnnz_gpu {
namespace {
using namespace sym;

constexpr int kHB = 256;                       // block of the unit passes
constexpr int kRunBlock = 1024;                // block of the task runners
constexpr int kHashSlots = 49152;              // 192 KB hash table
constexpr int64_t kHashTaskProducts = kBin5Max;  // load <= 0.5
constexpr int64_t kBitmapTaskProducts = 131072;
constexpr int kMaxRanges = 2048;               // B.cols < 2^31, W = 2^20

struct HeavyTask {
    int32_t item;   // index in the batch
    int32_t slot;   // merge bitmap slot, or -1
    int32_t mode;   // 0: hash over a pbuf span, 1: bitmap over a pbuf span,
                    // 2: bitmap over the item's own product range (R == 1)
    int32_t range;  // column range of a bitmap task
    int64_t p0, p1;
};
static_assert(sizeof(HeavyTask) == 32, "task layout");

__device__ __forceinline__ const int32_t* heavy_list(const SymScratch& sc, int64_t first) {
    return sc.lists + int64_t(kHeavyBin) * sc.capacity + first;
}

// ---- batch bookkeeping: units, entry offsets, product offsets (1 block)
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

// ---- one block per item: product prefix over its entries, B-row starts
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

// Locates unit u: item index, and the item's product window [p0, p1).
struct Unit {
    int64_t item;
    long long p0, p1;
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

// Block-wide walk over products [p0, p1) of heavy item `item`, via its entry
// prefix (chunks of BLOCK entries staged in shared memory).  fn(keys, valid).
template <int BLOCK, typename Fn>
__device__ __forceinline__ void item_products(const SymArgs& g, const SymScratch& sc,
                                              int64_t first, int64_t item, long long p0,
                                              long long p1, long long* s_off, int64_t* s_b0,
                                              Fn&& fn) {
    const ItemRow it = item_row(g, heavy_list(sc, first)[item]);
    const int64_t L = it.a1 - it.a0;
    const int64_t* ep = sc.heavy_epre + sc.heavy_eoff[item];
    const int64_t* eb = sc.heavy_eb0 + sc.heavy_eoff[item];
    int64_t e0 = 0, e1 = L - 1;  // largest entry with ep[e] <= p0
    while (e0 < e1) {
        const int64_t mid = (e0 + e1 + 1) >> 1;
        if (ep[mid] <= p0) e0 = mid; else e1 = mid - 1;
    }
    for (int64_t e = e0;;) {
        const int n = static_cast<int>(L - e < BLOCK ? L - e : BLOCK);
        __syncthreads();  // previous chunk fully consumed
        if (threadIdx.x < n) {
            s_off[threadIdx.x] = ep[e + threadIdx.x];
            s_b0[threadIdx.x] = eb[e + threadIdx.x];
        }
        if (threadIdx.x == 0) s_off[n] = ep[e + n];
        __syncthreads();
        const long long q0 = p0 > s_off[0] ? p0 : s_off[0];
        const long long q1 = p1 < s_off[n] ? p1 : s_off[n];
        chunk_products<BLOCK / 32>(s_off, s_b0, n, q0, q1, g.bcol, fn);
        const bool done = s_off[n] >= p1 || e + n >= L;
        if (done) break;
        e += n;
    }
    __syncthreads();
}

// ---- 1. per-unit histogram over column ranges
__global__ void __launch_bounds__(kHB) k_heavy_count(SymArgs g, SymScratch sc, int64_t first,
                                                     int64_t count, int R, int wshift) {
    __shared__ long long s_off[kHB + 1];
    __shared__ int64_t s_b0[kHB];
    __shared__ int s_hist[kMaxRanges];
    const long long units = sc.heavy_meta[0];
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        const Unit un = find_unit(sc, count, u);
        for (int r = threadIdx.x; r < R; r += kHB) s_hist[r] = 0;
        item_products<kHB>(g, sc, first, un.item, un.p0, un.p1, s_off, s_b0,
                           [&](const int (&keys)[kUnroll], const bool (&valid)[kUnroll], long long) {
#pragma unroll
                               for (int k = 0; k < kUnroll; ++k)
                                   warp_bucket_add(s_hist, valid[k] ? (keys[k] >> wshift) : -1);
                           });
        long long* rc = sc.heavy_rc + un.item * R;
        for (int r = threadIdx.x; r < R; r += kHB)
            if (s_hist[r])
                atomicAdd(reinterpret_cast<unsigned long long*>(&rc[r]),
                          static_cast<unsigned long long>(s_hist[r]));
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
__global__ void __launch_bounds__(kHB) k_heavy_scatter(SymArgs g, SymScratch sc, int64_t first,
                                                       int64_t count, int R, int wshift) {
    __shared__ long long s_off[kHB + 1];
    __shared__ int64_t s_b0[kHB];
    extern __shared__ int4 s_dyn_keys[];
    // dynamic: keys[kHeavyUnitProducts] | base[R] (int64) | hist[R]
    int32_t* s_keys = reinterpret_cast<int32_t*>(s_dyn_keys);
    long long* s_base = reinterpret_cast<long long*>(s_keys + kHeavyUnitProducts);
    int* s_hist = reinterpret_cast<int*>(s_base + R);
    const long long units = sc.heavy_meta[0];
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        const Unit un = find_unit(sc, count, u);
        for (int r = threadIdx.x; r < R; r += kHB) s_hist[r] = 0;
        // stage the unit's products (product p -> slot p - p0) and count ranges
        item_products<kHB>(g, sc, first, un.item, un.p0, un.p1, s_off, s_b0,
                           [&](const int (&keys)[kUnroll], const bool (&valid)[kUnroll],
                               long long p) {
#pragma unroll
                               for (int k = 0; k < kUnroll; ++k) {
                                   if (valid[k]) s_keys[p + 32 * k - un.p0] = keys[k];
                                   warp_bucket_add(s_hist, valid[k] ? (keys[k] >> wshift) : -1);
                               }
                           });
        // reserve each range's slice of the bucket, then reuse s_hist as the
        // per-range cursor inside it
        long long* cur = sc.heavy_cur + un.item * R;
        for (int r = threadIdx.x; r < R; r += kHB) {
            const int c = s_hist[r];
            s_base[r] = c ? static_cast<long long>(atomicAdd(
                                reinterpret_cast<unsigned long long*>(&cur[r]),
                                static_cast<unsigned long long>(c)))
                          : 0;
            s_hist[r] = 0;
        }
        __syncthreads();
        const int n = static_cast<int>(un.p1 - un.p0);
        for (int i0 = 0; i0 < n; i0 += kHB) {
            const int i = i0 + threadIdx.x;
            const int key = i < n ? s_keys[i] : 0;
            const int r = i < n ? (key >> wshift) : -1;
            const int rank = warp_bucket_add(s_hist, r);
            if (i < n) sc.heavy_pbuf[s_base[r] + rank] = key;
        }
        __syncthreads();
    }
}

// ---- 4. tasks per item (one thread per item; appends with one atomic)
// Builds item i's task list; with out == nullptr it only counts.  Bitmap
// tasks of a range that needs more than one task share a merge slot.
__device__ int build_tasks(const SymScratch& sc, int64_t i, int R, HeavyTask* out) {
    const int32_t item = static_cast<int32_t>(i);
    int k = 0;
    auto bitmap = [&](int32_t range, long long p0, long long p1, int mode) {
        const long long parts = (p1 - p0 + kBitmapTaskProducts - 1) / kBitmapTaskProducts;
        int32_t slot = -1;
        if (out && parts > 1)
            slot = static_cast<int32_t>(
                atomicAdd(reinterpret_cast<unsigned long long*>(&sc.heavy_meta[4]), 1ULL));
        for (long long q = 0; q < parts; ++q, ++k) {
            if (!out) continue;
            const long long a = p0 + q * kBitmapTaskProducts;
            const long long b = a + kBitmapTaskProducts < p1 ? a + kBitmapTaskProducts : p1;
            out[k] = HeavyTask{item, slot, mode, range, a, b};
        }
    };
    if (R == 1) {  // whole row in one range, read from the B rows
        bitmap(0, 0, sc.heavy_foff[i + 1] - sc.heavy_foff[i], 2);
        return k;
    }
    const long long* rc = sc.heavy_rc + i * R;
    const long long end = sc.heavy_foff[i + 1];
    long long g0 = -1, g1 = -1;  // open hash group [g0, g1) of the product buffer
    auto flush = [&]() {
        if (g0 >= 0 && g1 > g0) {
            if (out) out[k] = HeavyTask{item, -1, 0, 0, g0, g1};
            ++k;
        }
        g0 = g1 = -1;
    };
    for (int r = 0; r < R; ++r) {
        const long long b0 = rc[r];
        const long long b1 = r + 1 < R ? rc[r + 1] : end;
        if (b1 == b0) continue;
        if (b1 - b0 > kHashTaskProducts) {
            flush();
            bitmap(r, b0, b1, 1);
        } else if (g0 >= 0 && b1 - g0 <= kHashTaskProducts) {
            g1 = b1;
        } else {
            flush();
            g0 = b0;
            g1 = b1;
        }
    }
    flush();
    return k;
}

__global__ void k_heavy_tasks(SymScratch sc, int64_t count, int R, int64_t task_cap) {
    const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (i >= count) return;
    const int n = build_tasks(sc, i, R, nullptr);
    const long long base = static_cast<long long>(atomicAdd(
        reinterpret_cast<unsigned long long*>(&sc.heavy_meta[3]), static_cast<unsigned long long>(n)));
    if (base + n > task_cap) __trap();  // host sizes task_cap to heavy_task_bound()
    build_tasks(sc, i, R, reinterpret_cast<HeavyTask*>(sc.heavy_tasks) + base);
}

// ---- 5. run the tasks: one block per task, sets in shared memory.  Hash
// tasks (192 KB table) and bitmap tasks (W-bit bitmap, <= 128 KB) run in two
// kernels so each gets 1024 threads per SM.
template <bool HASH>
__global__ void __launch_bounds__(kRunBlock) k_heavy_run(SymArgs g, SymScratch sc, int64_t first,
                                                         int32_t wwords, int wshift) {
    extern __shared__ int4 s_dyn[];
    uint32_t* s_set = reinterpret_cast<uint32_t*>(s_dyn);
    __shared__ long long s_off[kRunBlock + 1];
    __shared__ int64_t s_b0[kRunBlock];
    __shared__ long long s_red[kRunBlock / 32];
    const HeavyTask* tasks = reinterpret_cast<const HeavyTask*>(sc.heavy_tasks);
    const long long ntask = sc.heavy_meta[3];
    const int32_t* list = heavy_list(sc, first);
    long long acc = 0;
    for (long long ti = blockIdx.x; ti < ntask; ti += gridDim.x) {
        const HeavyTask t = tasks[ti];
        if ((t.mode == 0) != HASH) continue;  // the other kernel's task
        int cnt = 0;
        if (HASH) {
            int* table = reinterpret_cast<int*>(s_set);
            for (int k = threadIdx.x; k < kHashSlots; k += kRunBlock) table[k] = kEmpty;
            __syncthreads();
            for (long long p = t.p0 + threadIdx.x; p < t.p1; p += kRunBlock * kUnroll) {
                int keys[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const long long q = p + u * kRunBlock;
                    keys[u] = q < t.p1 ? __ldg(&sc.heavy_pbuf[q]) : kEmpty;
                }
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
                    if (keys[u] != kEmpty) cnt += hash_insert(table, kHashSlots, keys[u]);
            }
        } else {
            for (int k = threadIdx.x; k < wwords; k += kRunBlock) s_set[k] = 0u;
            __syncthreads();
            const uint32_t lo_mask = (1u << wshift) - 1u;  // column offset inside the range
            auto insert = [&](const int (&keys)[kUnroll], const bool (&valid)[kUnroll], long long) {
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
                    if (valid[u]) {
                        const uint32_t off = static_cast<uint32_t>(keys[u]) & lo_mask;
                        const uint32_t bit = 1u << (off & 31);
                        cnt += (atomicOr(&s_set[off >> 5], bit) & bit) ? 0 : 1;
                    }
            };
            if (t.mode == 1) {
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
                // shared range: the bits this task adds first are what counts
                __syncthreads();
                cnt = 0;
                uint32_t* gbm = sc.pool + int64_t(t.slot) * wwords;
                for (int k = threadIdx.x; k < wwords; k += kRunBlock) {
                    const uint32_t w = s_set[k];
                    if (w) cnt += __popc(w & ~atomicOr(&gbm[k], w));
                }
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
__global__ void k_heavy_clean(SymScratch sc, int32_t wwords) {
    const long long used = sc.heavy_meta[4] * wwords;
    for (long long i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < used;
         i += int64_t(gridDim.x) * blockDim.x)
        sc.pool[i] = 0u;
}

}  // namespace

HeavyGeometry heavy_geometry(int32_t bcols) {
    HeavyGeometry h;
    int shift = 5;
    while ((int64_t(1) << shift) < bcols && shift < 20) ++shift;
    h.wshift = shift;  // range width 2^shift bits (>= 32, <= 2^20)
    h.ranges = static_cast<int>((int64_t(bcols) + (int64_t(1) << shift) - 1) >> shift);
    if (h.ranges < 1) h.ranges = 1;
    h.wwords = static_cast<int32_t>((int64_t(1) << shift) / 32);
    return h;
}

int64_t heavy_task_bound(int64_t count, int64_t products, int ranges) {
    // hash groups: at most 2 per kHashTaskProducts of products plus one per
    // item; bitmap parts: one per kBitmapTaskProducts plus one per range
    return count * (ranges + 2) + 2 * (products / kHashTaskProducts + 1) +
           products / kBitmapTaskProducts + 1;
}

int64_t heavy_slot_bound(int64_t, int64_t products) {
    // a merge slot serves one range that needs >= 2 bitmap tasks
    return products / kBitmapTaskProducts + 1;
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
        cudaFuncSetAttribute(k_heavy_run<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kHashSlots * 4);
        cudaFuncSetAttribute(k_heavy_run<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (1 << 20) / 8);
        cudaFuncSetAttribute(k_heavy_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(kHeavyUnitProducts * 4 + kMaxRanges * 12));
        attr_done |= 1u << (dev & 31);
    }
    const HeavyGeometry geo = heavy_geometry(args.bcols);
    k_heavy_prep<<<1, 256, 0, stream>>>(args, s, first, count);
    k_heavy_entries<<<static_cast<unsigned>(count), 256, 0, stream>>>(args, s, first);
    const unsigned grid = static_cast<unsigned>(num_sms) * 8;
    if (geo.ranges > 1) {
        cudaMemsetAsync(s.heavy_rc, 0, sizeof(long long) * count * geo.ranges, stream);
        k_heavy_count<<<grid, kHB, 0, stream>>>(args, s, first, count, geo.ranges, geo.wshift);
        k_heavy_offsets<<<static_cast<unsigned>((count + 255) / 256), 256, 0, stream>>>(
            s, count, geo.ranges);
        const int scatter_smem = int(kHeavyUnitProducts * 4 + geo.ranges * 12);
        k_heavy_scatter<<<static_cast<unsigned>(num_sms) * 6, kHB, scatter_smem, stream>>>(
            args, s, first, count, geo.ranges, geo.wshift);
    }
    k_heavy_tasks<<<static_cast<unsigned>((count + 127) / 128), 128, 0, stream>>>(
        s, count, geo.ranges, s.heavy_task_cap);
    if (geo.ranges > 1)
        k_heavy_run<true><<<static_cast<unsigned>(num_sms), kRunBlock, kHashSlots * 4, stream>>>(
            args, s, first, geo.wwords, geo.wshift);
    k_heavy_run<false><<<static_cast<unsigned>(num_sms), kRunBlock, geo.wwords * 4, stream>>>(
        args, s, first, geo.wwords, geo.wshift);
    k_heavy_clean<<<static_cast<unsigned>(num_sms) * 4, 256, 0, stream>>>(s, geo.wwords);
    return cudaGetLastError();
}

}  // namespace spnnz_gpu
