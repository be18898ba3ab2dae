// Symbolic SpGEMM row-NNZ engine: exact distinct-column count of output rows
// of C = A*B, for a list of sampled rows (spnnz::sampled_symbolic,
// proj/include/spnnz/symbolic.hpp:122-154) or for every row
// (spnnz::exact_symbolic, :94-118).  The reference probes one open-addressing
// table per thread (HashAccumulator::row_nnz, :35-60); the count it returns is
// a set cardinality, independent of the hash (proj/tests/test_symbolic.cpp:
// 94-109), so every tier below is free to pick its own set representation.
//
// Rows are binned by their FLOP (the table size the reference uses):
//   bin 1  f <= 32      one warp per row: products staged in registers,
//                       duplicates found with __match_any_sync
//   bin 2  f <= 512     one warp per row, 1024-slot shared-memory hash
//   bin 3  f <= 4096    256-thread block, 8192-slot shared-memory hash
//   bin 4  f <= 32768   512-thread block, 53248-slot shared-memory hash
//   bin 5  heavier      many blocks per row over a global-memory bitmap of
//                       B.cols bits, cleaned after use by re-walking products
// Products of a row chunk are enumerated flat: a block scan of the chunk's B
// row lengths gives offsets, each thread takes product p and finds its entry
// by binary search in shared memory, so consecutive threads read consecutive
// B.col addresses (coalesced) whatever the B row lengths are.
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

// ------------------------------------------------------------- binning
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_sym_bin(SymArgs g, SymScratch sc) {
    __shared__ long long s_red[BLOCK / 32];
    const int lane = threadIdx.x & 31;
    long long fsum = 0;
    const int64_t stride = int64_t(gridDim.x) * BLOCK;
    for (int64_t base = int64_t(blockIdx.x) * BLOCK; base < g.n_items; base += stride) {
        const int64_t s = base + threadIdx.x;
        int bin = 7;  // 7: not an item of this thread
        if (s < g.n_items) {
            const int32_t rid = g.rows ? g.rows[s] : g.row_lo + static_cast<int32_t>(s);
            const int32_t r = rid - g.row_lo;
            if (r >= 0 && r < g.a.rows) {
                const int64_t f = g.flop[r];
                fsum += f;
                bin = f == 0 ? 0 : f <= kBin1Max ? 1 : f <= kBin2Max ? 2 : f <= kBin3Max ? 3
                                 : f <= kBin4Max ? 4 : 5;
            } else {
                bin = 6;  // foreign row (another rank's shard)
            }
            if (g.out && (bin == 0 || bin == 5 || bin == 6)) g.out[s] = 0;
        }
        // total entries of heavy rows (sizes the per-entry prefix arrays)
        long long hl = 0;
        if (bin == 5) {
            const int32_t r = (g.rows ? g.rows[s] : g.row_lo + static_cast<int32_t>(s)) - g.row_lo;
            hl = g.a.rpt[r + 1] - g.a.rpt[r] + 1;
        }
        if (__any_sync(kFull, hl != 0)) {
            hl = warp_sum_ll(hl);
            if (lane == 0)
                atomicAdd(reinterpret_cast<unsigned long long*>(&sc.heavy_meta[1]),
                          static_cast<unsigned long long>(hl));
        }
        // warp-aggregated append to the bin lists
        const unsigned peers = __match_any_sync(kFull, bin);
        if (bin >= 1 && bin <= 5) {
            const int leader = __ffs(peers) - 1;
            int pos = 0;
            if (lane == leader) pos = atomicAdd(&sc.counts[bin], __popc(peers));
            pos = __shfl_sync(peers, pos, leader);
            pos += __popc(peers & ((1u << lane) - 1));
            sc.lists[int64_t(bin) * sc.capacity + pos] = static_cast<int32_t>(s);
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
            off[lane] = incl - d;
            b0s[lane] = b0;
            if (lane == 31) off[32] = incl;
            __syncwarp();
            const int P = off[32];
            for (int p = lane; p < P; p += 32) {
                int lo = 0, hi = 31;  // largest j with off[j] <= p
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (off[mid] <= p) lo = mid; else hi = mid - 1;
                }
                const int key = __ldg(&g.bcol[b0s[lo] + (p - off[lo])]);
                cnt += hash_insert(table, kSlots, key);
            }
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

// Block-cooperative enumeration of the products of entries [e_begin, e_end)
// of one A row, in chunks of BLOCK entries; fn(key) is called once per
// product by some thread.  Requires all threads of the block.
template <int BLOCK, typename Fn>
__device__ __forceinline__ void block_products(const SymArgs& g, int64_t e_begin, int64_t e_end,
                                               int* s_off /*BLOCK+1*/, int64_t* s_b0 /*BLOCK*/,
                                               Fn&& fn) {
    using Scan = cub::BlockScan<int, BLOCK>;
    __shared__ typename Scan::TempStorage scan_tmp;
    for (int64_t c0 = e_begin; c0 < e_end; c0 += BLOCK) {
        const int64_t e = c0 + threadIdx.x;
        int d = 0;
        int64_t b0 = 0;
        if (e < e_end) {
            const int c = __ldg(&g.a.col[e]);
            b0 = __ldg(&g.brpt[c]);
            d = static_cast<int>(__ldg(&g.brpt[c + 1]) - b0);
        }
        int excl, total;
        Scan(scan_tmp).ExclusiveSum(d, excl, total);
        s_off[threadIdx.x] = excl;
        s_b0[threadIdx.x] = b0;
        if (threadIdx.x == 0) s_off[BLOCK] = total;
        __syncthreads();
        const int nent = static_cast<int>(e_end - c0 < BLOCK ? e_end - c0 : BLOCK);
        for (int p = threadIdx.x; p < total; p += BLOCK) {
            int lo = 0, hi = nent - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_off[mid] <= p) lo = mid; else hi = mid - 1;
            }
            fn(__ldg(&g.bcol[s_b0[lo] + (p - s_off[lo])]));
        }
        __syncthreads();
    }
}

// ------------------------------ bins 3, 4: block + shared-memory hash
template <int BLOCK, int SLOTS, int BIN>
__global__ void __launch_bounds__(BLOCK) k_sym_block_hash(SymArgs g, SymScratch sc) {
    extern __shared__ int4 s_dyn[];
    int* table = reinterpret_cast<int*>(s_dyn);
    __shared__ int s_off[BLOCK + 1];
    __shared__ int64_t s_b0[BLOCK];
    __shared__ long long s_red[BLOCK / 32];
    const int32_t* list = sc.lists + int64_t(BIN) * sc.capacity;
    const int n = sc.counts[BIN];
    long long acc = 0;
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const ItemRow it = item_row(g, list[i]);
        for (int k = threadIdx.x; k < SLOTS; k += BLOCK) table[k] = kEmpty;
        __syncthreads();
        int cnt = 0;
        block_products<BLOCK>(g, it.a0, it.a1, s_off, s_b0,
                              [&](int key) { cnt += hash_insert(table, SLOTS, key); });
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

// ------------------------------------------------ bin 5: heavy rows
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
    const int32_t* list = sc.lists + 5 * sc.capacity + first;
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
    const ItemRow it = item_row(g, sc.lists[5 * sc.capacity + first + i]);
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
    __shared__ long long s_off[kHeavyBlock];
    __shared__ int64_t s_b0[kHeavyBlock];
    __shared__ long long s_end;
    __shared__ long long s_red[kHeavyBlock / 32];
    const int32_t* list = sc.lists + 5 * sc.capacity + first;
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
            if (threadIdx.x == 0) s_end = ep[e + n];
            __syncthreads();
            const long long q0 = p0 > s_off[0] ? p0 : s_off[0];
            const long long q1 = p1 < s_end ? p1 : s_end;
            for (long long p = q0 + threadIdx.x; p < q1; p += kHeavyBlock) {
                int jl = 0, jh = n - 1;
                while (jl < jh) {
                    const int mid = (jl + jh + 1) >> 1;
                    if (s_off[mid] <= p) jl = mid; else jh = mid - 1;
                }
                const int key = __ldg(&g.bcol[s_b0[jl] + (p - s_off[jl])]);
                uint32_t* w = bm + (static_cast<uint32_t>(key) >> 5);
                if (CLEAN) {
                    *w = 0u;
                } else {
                    const uint32_t bit = 1u << (key & 31);
                    if (!(*reinterpret_cast<volatile uint32_t*>(w) & bit))
                        cnt += (atomicOr(w, bit) & bit) ? 0 : 1;
                }
            }
            const bool done = s_end >= p1 || e + n >= L;
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

constexpr int kT3Block = 256, kT3Slots = 8192;
constexpr int kT4Block = 512, kT4Slots = 53248;

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
                             cudaStream_t stream) {
    if (args.n_items == 0) return cudaSuccess;
    static unsigned attr_done = 0;  // one bit per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_done & (1u << (dev & 31)))) {
        cudaFuncSetAttribute(k_sym_block_hash<kT3Block, kT3Slots, 3>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kT3Slots * 4);
        cudaFuncSetAttribute(k_sym_block_hash<kT4Block, kT4Slots, 4>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kT4Slots * 4);
        attr_done |= 1u << (dev & 31);
    }
    const unsigned g = static_cast<unsigned>(num_sms) * 4;
    k_sym_tiny<256><<<g, 256, 0, stream>>>(args, s);
    k_sym_warp_hash<256><<<g, 256, 0, stream>>>(args, s);
    k_sym_block_hash<kT3Block, kT3Slots, 3><<<g, kT3Block, kT3Slots * 4, stream>>>(args, s);
    k_sym_block_hash<kT4Block, kT4Slots, 4><<<static_cast<unsigned>(num_sms), kT4Block,
                                              kT4Slots * 4, stream>>>(args, s);
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
