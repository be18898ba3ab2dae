// Symbolic SpGEMM row-NNZ engine: exact distinct-column count of output rows
// of C = A*B, for a list of sampled rows (spnnz::sampled_symbolic,
// proj/include/spnnz/symbolic.hpp:122-154) or for every row
// (spnnz::exact_symbolic, :94-118).  The reference probes one open-addressing
// table per thread (HashAccumulator::row_nnz, :35-60); the count it returns is
// a set cardinality, independent of the hash (proj/tests/test_symbolic.cpp:
// 94-109), so every tier below is free to pick its own set representation.
//
// Rows are binned by their FLOP f (the reference's table size):
//   bin 1  f <= 32      one warp per row: products staged in registers,
//                       duplicates found with __match_any_sync
//   bin 2  f <= 512     one warp per row, 1024-slot shared-memory hash
//   bin 3  f <= 2048    256-thread block, 4096-slot shared-memory hash
//   bin 4  f <= 8192    512-thread block, 16384-slot shared-memory hash
//   bin 5  f <= 32768   512-thread block, 53248-slot shared-memory hash
//   bin 6  heavier      products split into 16 K-product units over the whole
//                       GPU, global-memory bitmap of B.cols bits per row,
//                       cleaned after use by re-walking the products
// Products are enumerated per chunk of entries: a scan of the chunk's B row
// lengths gives product offsets; each warp takes a contiguous slice of the
// chunk's products and its lanes walk them 32 apart with a monotone entry
// cursor, so a warp's loads of B.col are consecutive (coalesced) whatever the
// B row lengths, and each product costs ~1 shared-memory probe to locate.
#include <cub/block/block_scan.cuh>

#include "device_common.cuh"
#include "kernels.h"

namespace spnnz_gpu {
namespace {

constexpr int kEmpty = -1;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Open-addressing insert; returns 1 if key was new.  `size` slots, hash by
// multiply-high range reduction so any table size works.
__device__ __forceinline__ int hash_insert(int* table, uint32_t size, int key) {
    uint32_t h = __umulhi(mix32(static_cast<uint32_t>(key)), size);
    for (;;) {
        const int cur = table[h];
        if (cur == key) return 0;
        if (cur == kEmpty) {
            const int prev = atomicCAS(&table[h], kEmpty, key);
            if (prev == kEmpty) return 1;
            if (prev == key) return 0;
        }
        h = (h + 1 == size) ? 0 : h + 1;
    }
}

struct ItemRow {
    int64_t a0, a1;  // absolute nonzero range of the A row
    int32_t s;       // item index
};

__device__ __forceinline__ ItemRow item_row(const SymArgs& g, int32_t s) {
    const int32_t rid = g.rows ? g.rows[s] : g.row_lo + s;
    const int32_t r = rid - g.row_lo;
    ItemRow it;
    it.s = s;
    it.a0 = g.a.rpt[r];
    it.a1 = g.a.rpt[r + 1];
    return it;
}

// Walks products [q0, q1) of a chunk of n entries with exclusive offsets
// off[0..n] (off[n] = chunk end) and B-row starts b0[0..n).  WARPS warps
// share the range.  Each lane gathers kUnroll keys (32 apart) back to back
// and hands them to fn(keys, valid) together, so the loads -- and whatever
// memory operations fn issues per key -- overlap instead of forming one
// dependent chain per product.
constexpr int kUnroll = 4;

template <int WARPS, typename OffT, typename Fn>
__device__ __forceinline__ void chunk_products(const OffT* off, const int64_t* b0, int n,
                                               long long q0, long long q1,
                                               const int32_t* __restrict__ bcol, Fn&& fn) {
    const int lane = threadIdx.x & 31, w = (threadIdx.x >> 5) % WARPS;
    const long long span = q1 - q0;
    if (span <= 0 || n <= 0) return;
    long long per = (span + WARPS - 1) / WARPS;
    per = (per + 31) & ~31LL;
    const long long ws = q0 + w * per;
    const long long we = ws + per < q1 ? ws + per : q1;
    long long p = ws + lane;
    if (p >= we) return;
    int lo = 0, hi = n - 1;  // largest e with off[e] <= p
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (static_cast<long long>(off[mid]) <= p) lo = mid; else hi = mid - 1;
    }
    int e = lo;
    for (; p < we; p += 32 * kUnroll) {
        int keys[kUnroll];
        bool valid[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const long long q = p + 32 * u;
            valid[u] = q < we;
            keys[u] = 0;
            if (valid[u]) {
                while (static_cast<long long>(off[e + 1]) <= q) ++e;
                keys[u] = __ldg(&bcol[b0[e] + (q - static_cast<long long>(off[e]))]);
            }
        }
        fn(keys, valid);
    }
}

// fn adaptor: insert each valid key into a shared-memory hash table.
struct HashSink {
    int* table;
    uint32_t size;
    int* cnt;
    __device__ __forceinline__ void operator()(const int (&keys)[kUnroll],
                                               const bool (&valid)[kUnroll]) const {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            if (valid[u]) *cnt += hash_insert(table, size, keys[u]);
    }
};

// ------------------------------------------------------------- binning
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_sym_bin(SymArgs g, SymScratch sc) {
    __shared__ long long s_red[BLOCK / 32];
    const int lane = threadIdx.x & 31;
    long long fsum = 0;
    const int64_t stride = int64_t(gridDim.x) * BLOCK;
    for (int64_t base = int64_t(blockIdx.x) * BLOCK; base < g.n_items; base += stride) {
        const int64_t s = base + threadIdx.x;
        int bin = kNoBin;
        long long hl = 0;
        if (s < g.n_items) {
            const int32_t rid = g.rows ? g.rows[s] : g.row_lo + static_cast<int32_t>(s);
            const int32_t r = rid - g.row_lo;
            if (r >= 0 && r < g.a.rows) {
                const int64_t f = g.flop[r];
                fsum += f;
                bin = f == 0 ? 0 : f <= kBin1Max ? 1 : f <= kBin2Max ? 2 : f <= kBin3Max ? 3
                                 : f <= kBin4Max ? 4 : f <= kBin5Max ? 5 : kHeavyBin;
                if (bin == kHeavyBin) hl = g.a.rpt[r + 1] - g.a.rpt[r] + 1;
            } else {
                bin = kForeignBin;  // another rank's shard
            }
            if (g.out && (bin == 0 || bin == kHeavyBin || bin == kForeignBin)) g.out[s] = 0;
        }
        // warp-aggregated append to the bin lists
        const unsigned peers = __match_any_sync(kFull, bin);
        if (bin >= 1 && bin <= kHeavyBin) {
            const int leader = __ffs(peers) - 1;
            int pos = 0;
            if (lane == leader) pos = atomicAdd(&sc.counts[bin], __popc(peers));
            pos = __shfl_sync(peers, pos, leader);
            pos += __popc(peers & ((1u << lane) - 1));
            sc.lists[int64_t(bin) * sc.capacity + pos] = static_cast<int32_t>(s);
        }
        // total entries (+1 each) of heavy rows: sizes the per-entry arrays
        if (__any_sync(kFull, hl != 0)) {
            hl = warp_sum_ll(hl);
            if (lane == 0)
                atomicAdd(reinterpret_cast<unsigned long long*>(&sc.heavy_meta[1]),
                          static_cast<unsigned long long>(hl));
        }
    }
    if (g.sampled_flop) {
        fsum = block_sum_ll<BLOCK>(fsum, s_red);
        if (threadIdx.x == 0 && fsum)
            atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[kFStar]),
                      static_cast<unsigned long long>(fsum));
    }
}

// -------------------------------------------------- bin 1: warp + match
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_sym_tiny(SymArgs g, SymScratch sc) {
    __shared__ int s_buf[BLOCK];  // 32 products per warp
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int* buf = s_buf + wib * 32;
    const int32_t* list = sc.lists + 1 * sc.capacity;
    const int n = sc.counts[1];
    long long acc = 0;
    for (int i = blockIdx.x * (BLOCK / 32) + wib; i < n; i += gridDim.x * (BLOCK / 32)) {
        const ItemRow it = item_row(g, list[i]);
        int pos = 0;
        for (int64_t e0 = it.a0; e0 < it.a1; e0 += 32) {
            const int64_t e = e0 + lane;
            int d = 0;
            int64_t b0 = 0;
            if (e < it.a1) {
                const int c = __ldg(&g.a.col[e]);
                b0 = __ldg(&g.brpt[c]);
                d = static_cast<int>(__ldg(&g.brpt[c + 1]) - b0);
            }
            const int incl = warp_incl_scan(d);
            const int excl = incl - d;
            for (int k = 0; k < d; ++k) buf[pos + excl + k] = __ldg(&g.bcol[b0 + k]);
            pos += __shfl_sync(kFull, incl, 31);
        }
        __syncwarp();
        const int key = lane < pos ? buf[lane] : -1 - lane;
        const unsigned m = __match_any_sync(kFull, key);
        const bool leader = lane < pos && (__ffs(m) - 1) == lane;
        const int cnt = __popc(__ballot_sync(kFull, leader));
        if (lane == 0) {
            if (g.out) g.out[it.s] = cnt;
            acc += cnt;
        }
        __syncwarp();
    }
    if (lane == 0 && acc)
        atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[g.total_slot]),
                  static_cast<unsigned long long>(acc));
}

// ------------------------------------------ bin 2: warp + 1024-slot hash
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_sym_warp_hash(SymArgs g, SymScratch sc) {
    constexpr int kSlots = 1024;
    constexpr int W = BLOCK / 32;
    __shared__ int s_table[W][kSlots];
    __shared__ int s_off[W][33];
    __shared__ int64_t s_b0[W][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int* table = s_table[wib];
    int* off = s_off[wib];
    int64_t* b0s = s_b0[wib];
    const int32_t* list = sc.lists + 2 * sc.capacity;
    const int n = sc.counts[2];
    long long acc = 0;
    for (int i = blockIdx.x * W + wib; i < n; i += gridDim.x * W) {
        const ItemRow it = item_row(g, list[i]);
        for (int k = lane; k < kSlots; k += 32) table[k] = kEmpty;
        int cnt = 0;
        for (int64_t e0 = it.a0; e0 < it.a1; e0 += 32) {
            const int64_t e = e0 + lane;
            int d = 0;
            int64_t b0 = 0;
            if (e < it.a1) {
                const int c = __ldg(&g.a.col[e]);
                b0 = __ldg(&g.brpt[c]);
                d = static_cast<int>(__ldg(&g.brpt[c + 1]) - b0);
            }
            const int incl = warp_incl_scan(d);
            const int nent = static_cast<int>(it.a1 - e0 < 32 ? it.a1 - e0 : 32);
            off[lane] = incl - d;
            b0s[lane] = b0;
            if (lane == nent - 1) off[nent] = incl;
            __syncwarp();
            chunk_products<1>(off, b0s, nent, 0, off[nent], g.bcol, HashSink{table, kSlots, &cnt});
            __syncwarp();
        }
        cnt = static_cast<int>(warp_sum_ll(cnt));
        if (lane == 0) {
            if (g.out) g.out[it.s] = cnt;
            acc += cnt;
        }
        __syncwarp();
    }
    if (lane == 0 && acc)
        atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[g.total_slot]),
                  static_cast<unsigned long long>(acc));
}

// ------------------------------ bins 3-5: block + shared-memory hash
template <int BLOCK, int SLOTS, int BIN>
__global__ void __launch_bounds__(BLOCK) k_sym_block_hash(SymArgs g, SymScratch sc) {
    extern __shared__ int4 s_dyn[];
    int* table = reinterpret_cast<int*>(s_dyn);
    using Scan = cub::BlockScan<int, BLOCK>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int s_off[BLOCK + 1];
    __shared__ int64_t s_b0[BLOCK];
    __shared__ long long s_red[BLOCK / 32];
    const int32_t* list = sc.lists + int64_t(BIN) * sc.capacity;
    const int n = sc.counts[BIN];
    long long acc = 0;
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const ItemRow it = item_row(g, list[i]);
        for (int k = threadIdx.x; k < SLOTS; k += BLOCK) table[k] = kEmpty;
        int cnt = 0;
        for (int64_t c0 = it.a0; c0 < it.a1; c0 += BLOCK) {
            const int64_t e = c0 + threadIdx.x;
            int d = 0;
            int64_t b0 = 0;
            if (e < it.a1) {
                const int c = __ldg(&g.a.col[e]);
                b0 = __ldg(&g.brpt[c]);
                d = static_cast<int>(__ldg(&g.brpt[c + 1]) - b0);
            }
            int excl, total;
            Scan(scan_tmp).ExclusiveSum(d, excl, total);
            const int nent = static_cast<int>(it.a1 - c0 < BLOCK ? it.a1 - c0 : BLOCK);
            s_off[threadIdx.x] = excl;
            s_b0[threadIdx.x] = b0;
            if (threadIdx.x == 0) s_off[nent] = total;
            __syncthreads();  // also orders the table fill before the inserts
            chunk_products<BLOCK / 32>(s_off, s_b0, nent, 0, total, g.bcol,
                                       HashSink{table, SLOTS, &cnt});
            __syncthreads();
        }
        const long long tot = block_sum_ll<BLOCK>(cnt, s_red);
        if (threadIdx.x == 0) {
            if (g.out) g.out[it.s] = tot;
            acc += tot;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && acc)
        atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[g.total_slot]),
                  static_cast<unsigned long long>(acc));
}

// ------------------------------------------------ bin 6: heavy rows
// A heavy row's products are split into units of kHeavyUnitProducts; one
// block per unit (grid-stride), so hub rows whose entries point at hub B rows
// spread over the whole GPU.  Sets are global bitmaps of B.cols bits from the
// pool (one per row of the batch); insertion = test, then atomicOr, counting
// bits this thread turned on.  A second pass over the same products stores 0
// to every touched word, which returns the pool to all-zero without a memset.
constexpr int kHeavyBlock = 256;

// One block: per-item entry offsets and unit counts for the batch.
__global__ void __launch_bounds__(256) k_heavy_prep(SymArgs g, SymScratch sc, int64_t first,
                                                    int64_t count) {
    using Scan = cub::BlockScan<long long, 256>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ long long s_carry_u, s_carry_e;
    if (threadIdx.x == 0) s_carry_u = s_carry_e = 0;
    __syncthreads();
    const int32_t* list = sc.lists + int64_t(kHeavyBin) * sc.capacity + first;
    for (int64_t b = 0; b < count; b += 256) {
        const int64_t i = b + threadIdx.x;
        long long units = 0, ents = 0;
        if (i < count) {
            const int32_t s = list[i];
            const int32_t rid = g.rows ? g.rows[s] : g.row_lo + s;
            const ItemRow it = item_row(g, s);
            const long long f = g.flop[rid - g.row_lo];
            units = (f + kHeavyUnitProducts - 1) / kHeavyUnitProducts;
            ents = it.a1 - it.a0 + 1;
        }
        long long ue, ee, ut, et;
        Scan(tmp).ExclusiveSum(units, ue, ut);
        __syncthreads();
        Scan(tmp).ExclusiveSum(ents, ee, et);
        if (i < count) {
            sc.heavy_unit_off[i] = s_carry_u + ue;
            sc.heavy_eoff[i] = s_carry_e + ee;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s_carry_u += ut;
            s_carry_e += et;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        sc.heavy_unit_off[count] = s_carry_u;
        sc.heavy_eoff[count] = s_carry_e;
        sc.heavy_meta[0] = s_carry_u;
    }
}

// One block per heavy item: exclusive product prefix over its entries and
// the start of each entry's B row.
__global__ void __launch_bounds__(256) k_heavy_entries(SymArgs g, SymScratch sc, int64_t first) {
    using Scan = cub::BlockScan<long long, 256>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ long long s_carry;
    const int64_t i = blockIdx.x;
    const ItemRow it = item_row(g, sc.lists[int64_t(kHeavyBin) * sc.capacity + first + i]);
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

template <bool CLEAN>
__global__ void __launch_bounds__(kHeavyBlock) k_heavy(SymArgs g, SymScratch sc, int64_t first,
                                                       int64_t count, int64_t words) {
    __shared__ long long s_off[kHeavyBlock + 1];
    __shared__ int64_t s_b0[kHeavyBlock];
    __shared__ long long s_red[kHeavyBlock / 32];
    const int32_t* list = sc.lists + int64_t(kHeavyBin) * sc.capacity + first;
    const long long units = sc.heavy_meta[0];
    long long acc = 0;
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t lo = 0, hi = count - 1;  // item owning unit u
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (sc.heavy_unit_off[mid] <= u) lo = mid; else hi = mid - 1;
        }
        const int32_t s = list[lo];
        const ItemRow it = item_row(g, s);
        const int64_t L = it.a1 - it.a0;
        const int64_t* ep = sc.heavy_epre + sc.heavy_eoff[lo];
        const int64_t* eb = sc.heavy_eb0 + sc.heavy_eoff[lo];
        const long long p0 = (u - sc.heavy_unit_off[lo]) * kHeavyUnitProducts;
        const long long ftot = ep[L];
        const long long p1 = p0 + kHeavyUnitProducts < ftot ? p0 + kHeavyUnitProducts : ftot;
        int64_t e0 = 0, e1 = L - 1;  // largest entry with ep[e] <= p0
        while (e0 < e1) {
            const int64_t mid = (e0 + e1 + 1) >> 1;
            if (ep[mid] <= p0) e0 = mid; else e1 = mid - 1;
        }
        uint32_t* bm = sc.pool + lo * words;
        int cnt = 0;
        for (int64_t e = e0;;) {
            const int n = static_cast<int>(L - e < kHeavyBlock ? L - e : kHeavyBlock);
            if (threadIdx.x < n) {
                s_off[threadIdx.x] = ep[e + threadIdx.x];
                s_b0[threadIdx.x] = eb[e + threadIdx.x];
            }
            if (threadIdx.x == 0) s_off[n] = ep[e + n];
            __syncthreads();
            const long long q0 = p0 > s_off[0] ? p0 : s_off[0];
            const long long q1 = p1 < s_off[n] ? p1 : s_off[n];
            chunk_products<kHeavyBlock / 32>(
                s_off, s_b0, n, q0, q1, g.bcol,
                [&](const int (&keys)[kUnroll], const bool (&valid)[kUnroll]) {
                    if (CLEAN) {
#pragma unroll
                        for (int u = 0; u < kUnroll; ++u)
                            if (valid[u]) bm[static_cast<uint32_t>(keys[u]) >> 5] = 0u;
                    } else {
                        // test all words first (independent loads), then
                        // atomically set the bits still missing
                        uint32_t cur[kUnroll];
#pragma unroll
                        for (int u = 0; u < kUnroll; ++u)
                            cur[u] = valid[u] ? *reinterpret_cast<volatile uint32_t*>(
                                                    bm + (static_cast<uint32_t>(keys[u]) >> 5))
                                              : ~0u;
#pragma unroll
                        for (int u = 0; u < kUnroll; ++u) {
                            const uint32_t bit = 1u << (keys[u] & 31);
                            if (!(cur[u] & bit))
                                cnt += (atomicOr(bm + (static_cast<uint32_t>(keys[u]) >> 5), bit) &
                                        bit) ? 0 : 1;
                        }
                    }
                });
            const bool done = s_off[n] >= p1 || e + n >= L;
            __syncthreads();
            if (done) break;
            e += n;
        }
        if (!CLEAN) {
            const long long tot = block_sum_ll<kHeavyBlock>(cnt, s_red);
            if (threadIdx.x == 0 && tot) {
                if (g.out)
                    atomicAdd(reinterpret_cast<unsigned long long*>(&g.out[s]),
                              static_cast<unsigned long long>(tot));
                acc += tot;
            }
        }
        __syncthreads();
    }
    if (!CLEAN && threadIdx.x == 0 && acc)
        atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[g.total_slot]),
                  static_cast<unsigned long long>(acc));
}

constexpr int kT3Block = 256, kT3Slots = 4096;
constexpr int kT4Block = 512, kT4Slots = 16384;
constexpr int kT5Block = 512, kT5Slots = 53248;

template <int BLOCK, int SLOTS, int BIN>
void set_smem_attr() {
    cudaFuncSetAttribute(k_sym_block_hash<BLOCK, SLOTS, BIN>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, SLOTS * 4);
}

}  // namespace

int64_t heavy_table_words(int64_t, int32_t bcols) { return (int64_t(bcols) + 31) / 32; }

cudaError_t launch_sym_bin(const SymArgs& args, const SymScratch& s, cudaStream_t stream) {
    if (args.n_items == 0) return cudaSuccess;
    constexpr int B = 256;
    int64_t grid = (args.n_items + B - 1) / B;
    if (grid > 4096) grid = 4096;
    k_sym_bin<B><<<static_cast<unsigned>(grid), B, 0, stream>>>(args, s);
    return cudaGetLastError();
}

cudaError_t launch_sym_tiers(const SymArgs& args, const SymScratch& s, int num_sms,
                             const cudaStream_t* streams) {
    if (args.n_items == 0) return cudaSuccess;
    static unsigned attr_done = 0;  // one bit per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_done & (1u << (dev & 31)))) {
        set_smem_attr<kT3Block, kT3Slots, 3>();
        set_smem_attr<kT4Block, kT4Slots, 4>();
        set_smem_attr<kT5Block, kT5Slots, 5>();
        attr_done |= 1u << (dev & 31);
    }
    const unsigned sms = static_cast<unsigned>(num_sms);
    k_sym_tiny<256><<<sms * 4, 256, 0, streams[0]>>>(args, s);
    k_sym_warp_hash<256><<<sms * 4, 256, 0, streams[1]>>>(args, s);
    k_sym_block_hash<kT3Block, kT3Slots, 3><<<sms * 8, kT3Block, kT3Slots * 4, streams[2]>>>(args, s);
    k_sym_block_hash<kT4Block, kT4Slots, 4><<<sms * 3, kT4Block, kT4Slots * 4, streams[3]>>>(args, s);
    k_sym_block_hash<kT5Block, kT5Slots, 5><<<sms, kT5Block, kT5Slots * 4, streams[0]>>>(args, s);
    return cudaGetLastError();
}

cudaError_t launch_sym_heavy(const SymArgs& args, const SymScratch& s, int64_t first,
                             int64_t count, int num_sms, cudaStream_t stream) {
    if (count == 0) return cudaSuccess;
    const int64_t words = heavy_table_words(0, args.bcols);
    k_heavy_prep<<<1, 256, 0, stream>>>(args, s, first, count);
    k_heavy_entries<<<static_cast<unsigned>(count), 256, 0, stream>>>(args, s, first);
    const unsigned g = static_cast<unsigned>(num_sms) * 8;
    k_heavy<false><<<g, kHeavyBlock, 0, stream>>>(args, s, first, count, words);
    k_heavy<true><<<g, kHeavyBlock, 0, stream>>>(args, s, first, count, words);
    return cudaGetLastError();
}

}  // namespace spnnz_gpu
