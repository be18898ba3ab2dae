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
//   bin 5  f <= 24576   1024-thread block, 49152-slot shared-memory hash
//   bin 6  heavier      heavy.cu: products bucketed by column range, every
//                       set operation in shared memory, many blocks per row
// Products are enumerated per chunk of entries: a scan of the chunk's B row
// lengths gives product offsets; each warp takes a contiguous slice of the
// chunk's products and its lanes walk them 32 apart with a monotone entry
// cursor, so a warp's loads of B.col are consecutive (coalesced) whatever the
// B row lengths, and each product costs ~1 shared-memory probe to locate.
#include <atomic>

#include "symbolic_common.cuh"

namespace spnnz_gpu {
namespace {
using namespace sym;

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
        long long hl = 0, hf = 0, hb = 0, hp = 0;
        if (s < g.n_items) {
            const int32_t rid = g.rows ? g.rows[s] : g.row_lo + static_cast<int32_t>(s);
            const int32_t r = rid - g.row_lo;
            const bool mine = !g.window || (s >= g.window[0] && s < g.window[1]);
            if (mine && r >= 0 && r < g.a.rows) {
                const int64_t f = g.item_flop ? g.item_flop[s] : g.flop[r];
                const int64_t ts = g.tsize ? g.tsize[r] : f;  // the reference's table size
                fsum += ts;
                if (g.tsize && ts > g.tsize_cap)  // HashAccumulator: tsize exceeds capacity
                    atomicMax(reinterpret_cast<unsigned long long*>(&sc.heavy_meta[kMetaCapacity]),
                              static_cast<unsigned long long>(ts));
                bin = (f == 0 || ts == 0) ? 0 : f <= kBin1Max ? 1 : f <= kBin2Max ? 2 : f <= kBin3Max ? 3
                                 : f <= kBin4Max ? 4 : f <= kBin5Max ? 5 : f <= g.mp_max ? kMpBin : kHeavyBin;
                if (bin == kHeavyBin) {
                    hl = g.a.rpt[r + 1] - g.a.rpt[r] + 1;
                    hf = f;
                    hp = interval_geometry(g.bcols).count;
                    hb = (hp - 1) * (hl - 1);
                }
            } else {
                bin = kForeignBin;  // another rank's shard
            }
            if (g.out && (bin == 0 || bin == kHeavyBin || bin == kForeignBin)) g.out[s] = 0;
        }
        // warp-aggregated append to the bin lists
        const unsigned peers = __match_any_sync(kFull, bin);
        if ((bin >= 1 && bin <= kHeavyBin) || bin == kMpBin) {
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
            hf = warp_sum_ll(hf);
            hb = warp_sum_ll(hb);
            hp = warp_sum_ll(hp);
            if (lane == 0) {
                auto* m = reinterpret_cast<unsigned long long*>(sc.heavy_meta);
                atomicAdd(&m[1], static_cast<unsigned long long>(hl));
                atomicAdd(&m[2], static_cast<unsigned long long>(hf));
                atomicAdd(&m[5], static_cast<unsigned long long>(hb));
                atomicAdd(&m[6], static_cast<unsigned long long>(hp));
            }
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
    __shared__ __align__(16) int s_table[W][kSlots];
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
        hash_clear(table, kSlots, lane, 32);
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

// ------------------------------------ small problems: one fused kernel
// Every row's FLOP is at most kBin2Max (the context's own resident profile
// says so): no binning pass, no tier streams -- one warp per item draws its
// row (make_sample_plan's draw, as k_sample), walks its products into a
// 1024-slot shared hash (bin 2's tier), and adds the row's FLOP (f*, summed
// from the same walk) and its distinct count (z*).  A sampled call becomes
// one kernel instead of sample + bin + five tiers on four streams.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_sym_small(SymArgs g, uint64_t seed, int32_t num_rows, int draw,
                                                     int32_t* __restrict__ rows_out, int split) {
    constexpr int kSlots = 1024;
    constexpr int W = BLOCK / 32;
    __shared__ __align__(16) int s_table[W][kSlots];
    __shared__ int s_off[W][33];
    __shared__ int64_t s_b0[W][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int* table = s_table[wib];
    int* off = s_off[wib];
    int64_t* b0s = s_b0[wib];
    long long acc = 0, facc = 0;
    for (int64_t i = blockIdx.x * int64_t(W) + wib; i < g.n_items; i += int64_t(gridDim.x) * W) {
        int32_t rid;
        if (draw) {
            rid = draw_row(seed, static_cast<uint64_t>(i), num_rows);
            if (lane == 0) rows_out[i] = rid;
        } else {
            rid = g.rows[i];
        }
        const int32_t r = rid - g.row_lo;
        if (split && g.flop[r] > kBin2Max) continue;  // k_sym_small_block's (the resident own profile)
        const int64_t a0 = g.a.rpt[r], a1 = g.a.rpt[r + 1];
        hash_clear(table, kSlots, lane, 32);
        int cnt = 0;
        long long f = 0;
        for (int64_t e0 = a0; e0 < a1; e0 += 32) {
            const int64_t e = e0 + lane;
            int d = 0;
            int64_t b0 = 0;
            if (e < a1) {
                const int c = __ldg(&g.a.col[e]);
                b0 = __ldg(&g.brpt[c]);
                d = static_cast<int>(__ldg(&g.brpt[c + 1]) - b0);
            }
            f += d;
            const int incl = warp_incl_scan(d);
            const int nent = static_cast<int>(a1 - e0 < 32 ? a1 - e0 : 32);
            off[lane] = incl - d;
            b0s[lane] = b0;
            if (lane == nent - 1) off[nent] = incl;
            __syncwarp();
            chunk_products<1>(off, b0s, nent, 0, off[nent], g.bcol, HashSink{table, kSlots, &cnt});
            __syncwarp();
        }
        cnt = static_cast<int>(warp_sum_ll(cnt));
        f = warp_sum_ll(f);
        if (lane == 0) {
            if (g.out) g.out[i] = cnt;
            acc += cnt;
            facc += f;
        }
        __syncwarp();
    }
    if (lane == 0) {
        if (acc)
            atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[g.total_slot]),
                      static_cast<unsigned long long>(acc));
        if (g.sampled_flop && facc)
            atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[kFStar]), static_cast<unsigned long long>(facc));
    }
}

// The same for the items of kBin2Max < FLOP <= kBin3Max (launched beside
// k_sym_small when the profile's max is above bin 2): one block per item,
// bin 3's 4096-slot table, the item's row drawn again (the same draw).
template <int BLOCK, int SLOTS>
__global__ void __launch_bounds__(BLOCK) k_sym_small_block(SymArgs g, uint64_t seed, int32_t num_rows, int draw) {
    __shared__ __align__(16) int table[SLOTS];
    using Scan = cub::BlockScan<int, BLOCK>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int s_off[BLOCK + 1];
    __shared__ int64_t s_b0[BLOCK];
    __shared__ long long s_red[BLOCK / 32];
    long long acc = 0, facc = 0;
    for (int64_t i = blockIdx.x; i < g.n_items; i += gridDim.x) {
        const int32_t rid = draw ? draw_row(seed, static_cast<uint64_t>(i), num_rows) : g.rows[i];
        const int32_t r = rid - g.row_lo;
        const int64_t f = g.flop[r];
        if (f <= kBin2Max) continue;  // k_sym_small's (uniform per block)
        const int64_t a0 = g.a.rpt[r], a1 = g.a.rpt[r + 1];
        hash_clear(table, SLOTS, threadIdx.x, BLOCK);
        int cnt = 0;
        for (int64_t c0 = a0; c0 < a1; c0 += BLOCK) {
            const int64_t e = c0 + threadIdx.x;
            int d = 0;
            int64_t b0 = 0;
            if (e < a1) {
                const int c = __ldg(&g.a.col[e]);
                b0 = __ldg(&g.brpt[c]);
                d = static_cast<int>(__ldg(&g.brpt[c + 1]) - b0);
            }
            int excl, total;
            Scan(scan_tmp).ExclusiveSum(d, excl, total);
            const int nent = static_cast<int>(a1 - c0 < BLOCK ? a1 - c0 : BLOCK);
            s_off[threadIdx.x] = excl;
            s_b0[threadIdx.x] = b0;
            if (threadIdx.x == 0) s_off[nent] = total;
            __syncthreads();  // also orders the table fill before the inserts
            chunk_products<BLOCK / 32>(s_off, s_b0, nent, 0, total, g.bcol, HashSink{table, SLOTS, &cnt});
            __syncthreads();
        }
        const long long tot = block_sum_ll<BLOCK>(cnt, s_red);
        if (threadIdx.x == 0) {
            if (g.out) g.out[i] = tot;
            acc += tot;
            facc += f;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (acc)
            atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[g.total_slot]),
                      static_cast<unsigned long long>(acc));
        if (g.sampled_flop && facc)
            atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[kFStar]), static_cast<unsigned long long>(facc));
    }
}

// ------------------------------ bins 3-5: block + shared-memory hash
#ifndef SPNNZ_TIER_TICKETS
#define SPNNZ_TIER_TICKETS 1
#endif
static_assert(ticket_slot(3) > kNoBin && ticket_slot(kMpBin) < 16, "ticket counters live in the spare bin counters");
template <int BLOCK, int SLOTS, int BIN, int UNROLL>
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
    const uint32_t table_s = shared_window_reg(table);
    long long acc = 0;
#if SPNNZ_TIER_TICKETS
    // rows by ticket (counts[ticket_slot(BIN)], zeroed with the bin counts):
    // a bin's rows differ 3x in FLOP and a block sees only ~9-15 of them, so
    // static striding left the slowest block ~20-40 % over the mean.  Thread
    // 0 takes the next ticket while the current row runs (the L2 round trip
    // stays off the row's critical path).
    __shared__ int s_ticket;
    int next = 0;
    if (threadIdx.x == 0) next = atomicAdd(&sc.counts[ticket_slot(BIN)], 1);
    for (;;) {
        if (threadIdx.x == 0) s_ticket = next;
        __syncthreads();
        const int i = s_ticket;
        if (i >= n) break;
        if (threadIdx.x == 0) next = atomicAdd(&sc.counts[ticket_slot(BIN)], 1);
#else
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
#endif
        const ItemRow it = item_row(g, list[i]);
        hash_clear(table, SLOTS, threadIdx.x, BLOCK);
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
            chunk_products<BLOCK / 32, UNROLL>(s_off, s_b0, nent, 0, total, g.bcol,
                                               HashSinkU<UNROLL>{table, SLOTS, &cnt, table_s});
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

// ------------------------- multipass tier: kBin5Max < FLOP <= mp_max
// Bin 5's shape (one 1024-thread block per SM, a 49152-slot shared hash) for
// rows too big for one table: the row's products are walked P = ceil(FLOP /
// kMpPart) times and pass k inserts only the keys whose mixed hash lands in
// part k (mix32 is a bijection of the key, independent of the slot hash), so
// each pass sees ~FLOP / P products and the passes' distinct counts add up to
// the row's.  OPT-IN (SPNNZ_MP_MAX, default 0): the idea was that a filtered-
// out product costs only its coalesced load and one multiply, against the
// heavy path's counting sort + bitmap task (~190 thread instructions per
// product) -- but in SIMT a skipped key saves nothing while any lane of its
// warp inserts, so every pass costs bin 5's full ~3 warp instructions per
// product: measured 922 us for config 5's 45 M products of 24576 < FLOP <=
// 98304 (the heavy path: ~380 us for the same rows).  Kept under test as a
// recorded experiment.  Exactness does not depend on the hash: a pass whose table fills
// (probe sequence above kMpProbeCap -- keys crafted against mix32, or far
// more products in one part than the mean) raises a flag, and the row is
// redone with twice the passes; parts are hash ranges of a bijection, so
// that ends.  Rows of at most BLOCK entries (nearly all: FLOP <= 98304 at
// ~340 products per entry) stage their entry offsets once for all passes.
constexpr int kMpProbeCap = 2048;
__device__ __forceinline__ int hash_insert_shared_capped(uint32_t table_s, uint32_t size, int key) {
    uint32_t h = __umulhi(slot_hash(key), size);
    for (int probes = 0; probes < kMpProbeCap; ++probes) {
        const uint32_t addr = table_s + 4u * h;
        int cur;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(cur) : "r"(addr) : "memory");
        if (cur == key) return 0;
        if (cur == kEmpty) {
            int prev;
            asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;"
                         : "=r"(prev) : "r"(addr), "r"(kEmpty), "r"(key) : "memory");
            if (prev == kEmpty) return 1;
            if (prev == key) return 0;
        }
        h = (h + 1 == size) ? 0 : h + 1;
    }
    return -1;
}

template <int U>
struct PartSinkU {
    uint32_t table_s, size, part, parts;
    int* cnt;
    volatile int* ovf;
    __device__ __forceinline__ void operator()(const int (&keys)[U], const bool (&valid)[U], long long) const {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!valid[u] || __umulhi(mix32(static_cast<uint32_t>(keys[u])), parts) != part) continue;
            if (*ovf) continue;  // the pass is lost already: the row is redone
            const int r = hash_insert_shared_capped(table_s, size, keys[u]);
            if (r < 0) *ovf = 1; else *cnt += r;
        }
    }
};

template <int BLOCK, int SLOTS, int UNROLL>
__global__ void __launch_bounds__(BLOCK, 1) k_sym_multipass(SymArgs g, SymScratch sc) {
    extern __shared__ int4 s_dyn[];
    int* table = reinterpret_cast<int*>(s_dyn);
    using Scan = cub::BlockScan<int, BLOCK>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int s_off[BLOCK + 1];
    __shared__ int64_t s_b0[BLOCK];
    __shared__ long long s_red[BLOCK / 32];
    __shared__ int s_ticket, s_ovf;
    const int32_t* list = sc.lists + int64_t(kMpBin) * sc.capacity;
    const int n = sc.counts[kMpBin];
    const uint32_t table_s = static_cast<uint32_t>(__cvta_generic_to_shared(table));
    long long acc = 0;
    int next = 0;
    if (threadIdx.x == 0) next = atomicAdd(&sc.counts[ticket_slot(kMpBin)], 1);
    for (;;) {
        if (threadIdx.x == 0) s_ticket = next;
        __syncthreads();
        const int i = s_ticket;
        if (i >= n) break;
        if (threadIdx.x == 0) next = atomicAdd(&sc.counts[ticket_slot(kMpBin)], 1);
        const int32_t s = list[i];
        const ItemRow it = item_row(g, s);
        const int32_t rid = g.rows ? g.rows[s] : g.row_lo + s;
        const int64_t f = g.item_flop ? g.item_flop[s] : g.flop[rid - g.row_lo];
        uint32_t parts = static_cast<uint32_t>((f + g.mp_part - 1) / g.mp_part);
        if (parts < 1) parts = 1;
        const bool single = it.a1 - it.a0 <= BLOCK;  // one chunk of entries: staged once
        long long tot = 0;
        for (;;) {
            int cnt = 0;
            if (threadIdx.x == 0) s_ovf = 0;
            int nent = 0, total = 0;
            // entries [c0, c0 + BLOCK) -> s_off / s_b0 (every thread calls it)
#define SPNNZ_MP_STAGE(c0)                                                          \
    do {                                                                            \
        const int64_t e_ = (c0) + threadIdx.x;                                      \
        int d_ = 0;                                                                 \
        int64_t b0_ = 0;                                                            \
        if (e_ < it.a1) {                                                           \
            const int c_ = __ldg(&g.a.col[e_]);                                     \
            b0_ = __ldg(&g.brpt[c_]);                                               \
            d_ = static_cast<int>(__ldg(&g.brpt[c_ + 1]) - b0_);                    \
        }                                                                           \
        int excl_;                                                                  \
        Scan(scan_tmp).ExclusiveSum(d_, excl_, total);                              \
        nent = static_cast<int>(it.a1 - (c0) < BLOCK ? it.a1 - (c0) : BLOCK);       \
        s_off[threadIdx.x] = excl_;                                                 \
        s_b0[threadIdx.x] = b0_;                                                    \
        if (threadIdx.x == 0) s_off[nent] = total;                                  \
    } while (0)
            if (single) SPNNZ_MP_STAGE(it.a0);
            for (uint32_t part = 0; part < parts; ++part) {
                hash_clear(table, SLOTS, threadIdx.x, BLOCK);
                const PartSinkU<UNROLL> sink{table_s, static_cast<uint32_t>(SLOTS), part, parts, &cnt, &s_ovf};
                if (single) {
                    __syncthreads();  // the staged entries and the cleared table (and s_ovf = 0)
                    chunk_products<BLOCK / 32, UNROLL>(s_off, s_b0, nent, 0, total, g.bcol, sink);
                    __syncthreads();  // inserts done before the next pass clears
                } else {
                    for (int64_t c0 = it.a0; c0 < it.a1; c0 += BLOCK) {
                        SPNNZ_MP_STAGE(c0);
                        __syncthreads();
                        chunk_products<BLOCK / 32, UNROLL>(s_off, s_b0, nent, 0, total, g.bcol, sink);
                        __syncthreads();
                    }
                }
#undef SPNNZ_MP_STAGE
                if (s_ovf) break;  // uniform: read after the barrier that ends the pass
            }
            __syncthreads();
            const bool ovf = s_ovf != 0;
            tot = block_sum_ll<BLOCK>(cnt, s_red);
            __syncthreads();  // s_ovf and s_red are reused by a redo / the next row
            if (!ovf) break;
            parts *= 2;
        }
        if (threadIdx.x == 0) {
            if (g.out) g.out[it.s] = tot;
            acc += tot;
        }
    }
    if (threadIdx.x == 0 && acc)
        atomicAdd(reinterpret_cast<unsigned long long*>(&g.totals[g.total_slot]),
                  static_cast<unsigned long long>(acc));
}

#ifndef SPNNZ_T4_SLOTS
#define SPNNZ_T4_SLOTS 16384
#endif
#ifndef SPNNZ_T4_BLOCKS_PER_SM
#define SPNNZ_T4_BLOCKS_PER_SM 3
#endif
constexpr int kT3Block = 256, kT3Slots = 4096;
constexpr int kT4Block = 512, kT4Slots = SPNNZ_T4_SLOTS;
constexpr int kT5Block = 1024, kT5Slots = 49152;
// every shared hash table holds its bin's largest row at load <= 1/2, so a
// probe always finds an empty slot (the A/B build knobs SPNNZ_BIN*_MAX
// cannot push a row past its table: a full table would never terminate)
static_assert(1024 >= 2 * kBin2Max, "bin-2 table load <= 1/2");
static_assert(kT3Slots >= 2 * kBin3Max, "bin-3 table load <= 1/2");
static_assert(kT4Slots >= 2 * kBin4Max, "bin-4 table load <= 1/2");
static_assert(kT5Slots >= 2 * kBin5Max, "bin-5 table load <= 1/2");
static_assert(kBin1Max <= 32, "bin 1 stages a row's products in one warp's 32 slots");
// keys in flight per lane (B.col loads issued together before the inserts)
#ifndef SPNNZ_T3_UNROLL
#define SPNNZ_T3_UNROLL 4
#endif
#ifndef SPNNZ_T4_UNROLL
#define SPNNZ_T4_UNROLL 8
#endif
#ifndef SPNNZ_T5_UNROLL
#define SPNNZ_T5_UNROLL 8
#endif
#ifndef SPNNZ_MP_UNROLL
#define SPNNZ_MP_UNROLL 8
#endif

template <int BLOCK, int SLOTS, int BIN, int UNROLL>
void set_smem_attr() {
    cudaFuncSetAttribute(k_sym_block_hash<BLOCK, SLOTS, BIN, UNROLL>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, SLOTS * 4);
}

}  // namespace

cudaError_t launch_sym_small(const SymArgs& args, uint64_t seed, int32_t num_rows, bool draw, int32_t* rows_out,
                             int num_sms, cudaStream_t stream, cudaStream_t stream_b) {
    if (args.n_items == 0) return cudaSuccess;
    constexpr int B = 256;
    int64_t grid = (args.n_items + B / 32 - 1) / (B / 32);
    if (grid > int64_t(num_sms) * 8) grid = int64_t(num_sms) * 8;
    k_sym_small<B><<<static_cast<unsigned>(grid), B, 0, stream>>>(args, seed, num_rows, draw ? 1 : 0, rows_out,
                                                                    stream_b ? 1 : 0);
    if (stream_b) {
        int64_t gb = args.n_items < int64_t(num_sms) * 8 ? args.n_items : int64_t(num_sms) * 8;
        k_sym_small_block<256, 4096><<<static_cast<unsigned>(gb), 256, 0, stream_b>>>(args, seed, num_rows,
                                                                                     draw ? 1 : 0);
    }
    return cudaGetLastError();
}

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
    static std::atomic<unsigned long long> attr_done{0};  // one bit per device; the sets are idempotent
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_done.load(std::memory_order_acquire) & (1ull << (dev & 63)))) {
        set_smem_attr<kT3Block, kT3Slots, 3, SPNNZ_T3_UNROLL>();
        set_smem_attr<kT4Block, kT4Slots, 4, SPNNZ_T4_UNROLL>();
        set_smem_attr<kT5Block, kT5Slots, 5, SPNNZ_T5_UNROLL>();
        cudaFuncSetAttribute(k_sym_multipass<kT5Block, kT5Slots, SPNNZ_MP_UNROLL>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kT5Slots * 4);
        attr_done.fetch_or(1ull << (dev & 63), std::memory_order_release);
    }
    const unsigned sms = static_cast<unsigned>(num_sms);
    k_sym_tiny<256><<<sms * 4, 256, 0, streams[0]>>>(args, s);
    k_sym_warp_hash<256><<<sms * 4, 256, 0, streams[0]>>>(args, s);
    // grid multiple (A/B knob SPNNZ_TIER_WAVES): more, shorter blocks over
    // the same rows free SMs between rows (for higher-priority work)
    static const int waves = [] {
        const char* e = getenv("SPNNZ_TIER_WAVES");
        return e && atoi(e) > 0 ? atoi(e) : 1;
    }();
    k_sym_block_hash<kT3Block, kT3Slots, 3, SPNNZ_T3_UNROLL><<<sms * 8 * waves, kT3Block, kT3Slots * 4, streams[1]>>>(args, s);
    k_sym_block_hash<kT4Block, kT4Slots, 4, SPNNZ_T4_UNROLL><<<sms * SPNNZ_T4_BLOCKS_PER_SM * waves, kT4Block, kT4Slots * 4, streams[2]>>>(args, s);
    k_sym_block_hash<kT5Block, kT5Slots, 5, SPNNZ_T5_UNROLL><<<sms * waves, kT5Block, kT5Slots * 4, streams[3]>>>(args, s);
    // the multipass rows (bin 5's footprint: one block per SM) before bin 5 would
    // hold the biggest rows back; after it they share its stream
    if (args.mp_max > kBin5Max)
        k_sym_multipass<kT5Block, kT5Slots, SPNNZ_MP_UNROLL><<<sms, kT5Block, kT5Slots * 4, streams[3]>>>(args, s);
    return cudaGetLastError();
}

}  // namespace spnnz_gpu
