// Device-side helpers shared by the predictor kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace spnnz_gpu {

// Device-side bounds checks (a build with -DSPNNZ_DEBUG_BOUNDS=1; the GPU
// pool has compute-sanitizer closed): a violated index traps the kernel, so
// the call fails loudly instead of reading or writing past a table.
#ifndef SPNNZ_DEBUG_BOUNDS
#define SPNNZ_DEBUG_BOUNDS 0
#endif
#if SPNNZ_DEBUG_BOUNDS
#define SPNNZ_ASSERT(cond) \
    do {                  \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define SPNNZ_ASSERT(cond) \
    do {                  \
    } while (0)
#endif

constexpr int kWarp = 32;

// SplitMix64 output number r (0-based) of a generator seeded with `seed`:
// the reference advances state += gamma before mixing (rng.hpp:14-19), so
// draw r mixes seed + (r + 1) * gamma.  Counter-based => one thread per draw.
__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t r) {
    uint64_t z = seed + (r + 1) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// Row of draw r of make_sample_plan (predict.hpp:48-54): u = (z >> 11) 2^-53
// exact, M u one IEEE multiply, truncation toward zero, the rid >= M guard.
__device__ __forceinline__ int32_t draw_row(uint64_t seed, uint64_t r, int32_t num_rows) {
    const uint64_t z = splitmix_at(seed, r);
    const double u = __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53);
    const int32_t rid = __double2int_rz(__dmul_rn(static_cast<double>(num_rows), u));
    return rid >= num_rows ? num_rows - 1 : rid;
}

// 32-bit mixer for hash-table slots (any injective-enough mix works: the
// distinct count does not depend on the hash, symbolic.hpp:13-16 and
// proj/tests/test_symbolic.cpp:94-109).
__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

template <typename T>
__device__ __forceinline__ T ldg(const T* p) { return __ldg(p); }

// L2 eviction policies (createpolicy): streamed-once data is marked
// evict_first so it does not push the gathered arrays (B's degrees, B.col
// rows) out of the 126 MB L2; gathered data is marked evict_last.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int ld_stream_i32(const int* p, uint64_t pol) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
                 : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ long long ld_stream_i64(const long long* p, uint64_t pol) {
    long long v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;"
                 : "=l"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int4 ld_stream_v4(const int4* p, uint64_t pol) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int ld_keep_i32(const int* p, uint64_t pol) {
    int v;
    asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint16_t ld_keep_u16(const uint16_t* p, uint64_t pol) {
    unsigned short v;
    asm volatile("ld.global.nc.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_keep_u16(uint16_t* p, uint16_t v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.u16 [%0], %1, %2;" :: "l"(p), "h"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep_i32(int* p, int v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" :: "l"(p), "r"(v), "l"(pol) : "memory");
}

// Streaming 16-byte load that does not allocate in L1 (read-once data).
__device__ __forceinline__ longlong2 ld_stream_ll2(const longlong2* p) {
    longlong2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.s64 {%0, %1}, [%2];"
                 : "=l"(r.x), "=l"(r.y) : "l"(p));
    return r;
}

__device__ __forceinline__ void st_stream_ll2(longlong2* p, longlong2 v) {
    asm volatile("st.global.cs.v2.s64 [%0], {%1, %2};" :: "l"(p), "l"(v.x), "l"(v.y) : "memory");
}

__device__ __forceinline__ void st_stream_d2(double2* p, double2 v) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" :: "l"(p), "d"(v.x), "d"(v.y) : "memory");
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ long long warp_max_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

// Block-wide int64 sum/max of per-thread values.  The result is valid in
// warp 0 (callers use it from thread 0); the scratch may be reused by the
// next call (leading barrier).
template <int BLOCK>
__device__ __forceinline__ long long block_sum_ll(long long v, long long* scratch /* BLOCK/32 */) {
    v = warp_sum_ll(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) scratch[w] = v;
    __syncthreads();
    long long t = 0;
    if (w == 0) {
        t = l < BLOCK / 32 ? scratch[l] : 0;
        t = warp_sum_ll(t);
    }
    return t;
}

template <int BLOCK>
__device__ __forceinline__ long long block_max_ll(long long v, long long* scratch) {
    v = warp_max_ll(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) scratch[w] = v;
    __syncthreads();
    long long t = 0;
    if (w == 0) {
        t = l < BLOCK / 32 ? scratch[l] : 0;
        t = warp_max_ll(t);
    }
    return t;
}

// Predicted CR from the combined totals, exactly collect_sample_stats /
// predict_proposed (predict.hpp:86-89, :111-117): f*/z* in IEEE double, or 1.
__device__ __forceinline__ double predicted_cr(long long f_star, long long z_star) {
    return (f_star > 0 && z_star > 0) ? __ddiv_rn((double)f_star, (double)z_star) : 1.0;
}

// (int64)ceil(q) exactly as the reference's x86-64 build evaluates it: a
// quotient >= 2^63 (only for cr < 1 and huge rows) converts to the "integer
// indefinite" value INT64_MIN (cvttsd2si), where the GPU's cvt would saturate.
__device__ __forceinline__ long long ceil_of(long long f, double q) {
    const double cq = ceil(q);
    const long long c = cq >= 9223372036854775808.0 ? static_cast<long long>(0x8000000000000000ULL)
                                                    : static_cast<long long>(cq);
    return f < c ? f : c;
}

// Empty rows skip the division: 0 / cr is +0 for every accepted cr (> 0, +inf
// included; NaN is rejected at the boundary), and __ddiv_rn sends a zero
// dividend down its slow path (config 5: ~20 % empty rows, 72 -> 55 us for
// the pass, tools/microbench/predict_bw.cu).
__device__ __forceinline__ long long ceil_view(long long f, double cr, double* q_out) {
    if (f == 0) {
        *q_out = 0.0;
        return 0;
    }
    const double q = __ddiv_rn(static_cast<double>(f), cr);
    *q_out = q;
    return ceil_of(f, q);
}

// a / b correctly rounded (== __ddiv_rn) for a fixed divisor b >= 1 without
// a division per call: q from the reciprocal y = RN(1/b) plus one FMA
// correction, then an exact acceptance test -- the remainder r = a - q b is
// exact (FMA, q within an ulp), ulp(q) * b is exact (power-of-two scaling),
// and |r| < ulp(q) b / 2 means q is the unique nearest double to a / b.
// Anything else (ties, a <= 0) takes __ddiv_rn.
struct FastDiv {
    double b, y;
    __device__ __forceinline__ void init(double b_) {
        b = b_;
        y = __drcp_rn(b_);
    }
    // q = a / b correctly rounded when it returns true (a > 0, b >= 1); false
    // leaves the case to __ddiv_rn.
    __device__ __forceinline__ bool fast(double a, double* q_out) const {
        if (!(a > 0.0 && b >= 1.0)) return false;
        double q = __dmul_rn(a, y);
        q = __fma_rn(__fma_rn(-q, b, a), y, q);
        const double r = __fma_rn(-q, b, a);
        const double u = __longlong_as_double((__double_as_longlong(q) & 0x7ff0000000000000LL) -
                                              (52LL << 52));
        *q_out = q;
        return __dmul_rn(2.0, fabs(r)) < __dmul_rn(u, b);
    }
    __device__ __forceinline__ double operator()(double a) const {
        double q;
        return fast(a, &q) ? q : __ddiv_rn(a, b);
    }
};

}  // namespace spnnz_gpu
