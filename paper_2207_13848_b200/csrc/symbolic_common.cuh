// Device helpers shared by the symbolic tiers (symbolic.cu) and the heavy-row
// path (heavy.cu): item decoding, shared-memory hash insert and the
// coalesced product enumeration of a chunk of A-row entries.
#pragma once
#include <cub/block/block_scan.cuh>

#include "device_common.cuh"
#include "kernels.h"

namespace spnnz_gpu {
namespace sym {

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
#if SPNNZ_DEBUG_BOUNDS
    uint32_t probes = 0;
#endif
    for (;;) {
#if SPNNZ_DEBUG_BOUNDS
        SPNNZ_ASSERT(++probes <= size);  // a full table would never terminate
#endif
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
// and hands them to fn(keys, valid, p) together (keys[u] is product p+32u),
// so the loads -- and whatever
// memory operations fn issues per key -- overlap instead of forming one
// dependent chain per product.
#ifndef SPNNZ_UNROLL
#define SPNNZ_UNROLL 4
#endif
constexpr int kUnroll = SPNNZ_UNROLL;  // A/B: 8 -> config 5 step see DESIGN
#ifndef SPNNZ_CHUNK_FAST
#define SPNNZ_CHUNK_FAST 1
#endif

// A shared-memory pointer's 32-bit window address, opaque to the compiler so
// it stays in a register: left to itself the compiler re-derives the window
// (S2R SR_CgaCtaId + three more instructions) at every access in a loop.
__device__ __forceinline__ uint32_t shared_window_reg(const void* p) {
    uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    asm volatile("" : "+r"(a));
    return a;
}
__device__ __forceinline__ int lds_i32(uint32_t addr) {
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ long long lds_i64(uint32_t addr) {
    long long v;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
}

// off / b0 are SHARED-memory arrays (every caller stages them there): they are
// read through register-held window addresses, and the lane's current entry
// is kept as a pointer to its product 0 in bcol, so a key costs one 32 x 32 +
// 64 multiply-add for its address instead of a 64-bit add, a shift and the
// window derivation.
template <int WARPS, int U = kUnroll, typename Fn>
__device__ __forceinline__ void chunk_products(const int* off, const int64_t* b0, int n, int q0,
                                               int q1, const int32_t* __restrict__ bcol, Fn&& fn) {
    const int lane = threadIdx.x & 31, w = (threadIdx.x >> 5) % WARPS;
    const int span = q1 - q0;
    if (span <= 0 || n <= 0) return;
    const uint32_t off_s = shared_window_reg(off), b0_s = shared_window_reg(b0);
    int per = (span + WARPS - 1) / WARPS;
    per = (per + 31) & ~31;
    const int ws = q0 + w * per;
    const int we = ws + per < q1 ? ws + per : q1;
    // warp-uniform loop (fn may use warp collectives); lanes past the end of
    // the warp's slice run with valid = false
    int e = 0;
    if (ws + lane < we) {
        const int p = ws + lane;
        int lo = 0, hi = n - 1;  // largest e with off[e] <= p
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (lds_i32(off_s + 4u * mid) <= p) lo = mid; else hi = mid - 1;
        }
        e = lo;
    }
    // the lane's current entry lives in registers: its end offset and the
    // address of its product 0 in bcol (key of product q = bp[q])
    int nxt = lds_i32(off_s + 4u * (e + 1));
    const int32_t* bp = bcol + (lds_i64(b0_s + 8u * e) - static_cast<long long>(lds_i32(off_s + 4u * e)));
    const auto advance = [&](int q) {  // the lane's entry for product q >= nxt
        do {
            ++e;
            SPNNZ_ASSERT(e < n);
            nxt = lds_i32(off_s + 4u * (e + 1));
        } while (nxt <= q);
        bp = bcol + (lds_i64(b0_s + 8u * e) - static_cast<long long>(lds_i32(off_s + 4u * e)));
    };
    int base = ws;
#if SPNNZ_CHUNK_FAST
    // whole iterations (every lane's U products inside the slice): no range
    // checks, and fn sees constant-true valid flags (its per-key tests fold)
    for (; base + 32 * U <= we; base += 32 * U) {
        const int p = base + lane;
        int keys[U];
        bool valid[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int q = p + 32 * u;
            valid[u] = true;
            if (nxt <= q) advance(q);
            keys[u] = __ldg(bp + q);
        }
        fn(keys, valid, static_cast<long long>(p));
    }
#endif
    for (; base < we; base += 32 * U) {
        const int p = base + lane;
        int keys[U];
        bool valid[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int q = p + 32 * u;
            valid[u] = q < we;
            keys[u] = 0;
            if (valid[u]) {
                if (nxt <= q) advance(q);
                keys[u] = __ldg(bp + q);
            }
        }
        fn(keys, valid, static_cast<long long>(p));  // keys[u] is product p + 32 u
    }
}

// Warp-aggregated shared-memory add: lanes with the same bucket combine, the
// lowest of them adds; returns the lane's rank among its bucket peers plus
// the value the bucket had before (so it doubles as a cursor).  Must be
// called by all 32 lanes; bucket < 0 means "not participating".
__device__ __forceinline__ int warp_bucket_add(int* counters, int bucket) {
    const unsigned peers = __match_any_sync(0xffffffffu, bucket);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (bucket >= 0 && lane == leader) base = atomicAdd(&counters[bucket], __popc(peers));
    base = __shfl_sync(peers, base, leader);
    return base + __popc(peers & ((1u << lane) - 1));
}

// Fills a table with kEmpty using 16-byte stores (size a multiple of 4).
__device__ __forceinline__ void hash_clear(int* table, int size, int t, int nt) {
    int4* t4 = reinterpret_cast<int4*>(table);
    for (int k = t; k < (size >> 2); k += nt) t4[k] = make_int4(kEmpty, kEmpty, kEmpty, kEmpty);
}

#ifndef SPNNZ_HASH_PTX
#define SPNNZ_HASH_PTX 1
#endif
// hash_insert on a 32-bit shared-window address: the generic-pointer form
// re-derives the shared window (S2R SR_CgaCtaId + 64-bit arithmetic) on every
// probe of the loop.
#ifndef SPNNZ_HASH_FIB
#define SPNNZ_HASH_FIB 1
#endif
// slot hash: one Fibonacci multiply (default; config 5 step -13 us) or mix32 (A/B knob)
__device__ __forceinline__ uint32_t slot_hash(int key) {
#if SPNNZ_HASH_FIB
    return static_cast<uint32_t>(key) * 0x9E3779B1u;
#else
    return mix32(static_cast<uint32_t>(key));
#endif
}

__device__ __forceinline__ int hash_insert_shared(uint32_t table_s, uint32_t size, int key) {
    uint32_t h = __umulhi(slot_hash(key), size);
#if SPNNZ_DEBUG_BOUNDS
    uint32_t probes = 0;
#endif
    for (;;) {
#if SPNNZ_DEBUG_BOUNDS
        SPNNZ_ASSERT(++probes <= size);  // a full table would never terminate
#endif
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
}

// fn adaptor: insert each valid key into a shared-memory hash table.
template <int U = kUnroll>
struct HashSinkU {
    int* table;
    uint32_t size;
    int* cnt;
    // the table's shared-window address when the kernel holds it in a register
    // (shared_window_reg): derived from `table` per key otherwise
    uint32_t table_s = 0;
    __device__ __forceinline__ void operator()(const int (&keys)[U], const bool (&valid)[U], long long) const {
#if SPNNZ_HASH_PTX
        const uint32_t ts = table_s ? table_s : static_cast<uint32_t>(__cvta_generic_to_shared(table));
#endif
#pragma unroll
        for (int u = 0; u < U; ++u)
#if SPNNZ_HASH_PTX
            if (valid[u]) *cnt += hash_insert_shared(ts, size, keys[u]);
#else
            if (valid[u]) *cnt += hash_insert(table, size, keys[u]);
#endif
    }
};
using HashSink = HashSinkU<kUnroll>;

}  // namespace sym
}  // namespace spnnz_gpu
