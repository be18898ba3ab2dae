// Ceiling of the FLOP pass's access pattern on the real config-5 input.
//
// The FLOP pass (csrc/flop.cu) is one uint16 degree gather per A nonzero
// plus a stream of A.col.  This measures, on the same R-MAT 2^24 matrix
// (402.6 M nonzeros, built by libspnnz_gen exactly as bench.py does), the
// same loads with none of the pass's row logic:
//   stream : A.col only (16 consecutive columns per thread, 16-byte loads,
//            evict_first, L1-allocating -- the k_flop loads), summed;
//   gather : the same plus the 16 degree gathers (evict_last), summed;
// each thread writes one int64 so nothing is dead code.  The gather rate of
// "gather" is the most the FLOP pass can reach on this pattern on this part.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../../include -I../../paper_2207_13848_b200/csrc flop_ceiling.cu \
//        -L../../paper_2207_13848_b200/_lib -lspnnz_gen -o flop_ceiling
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "device_common.cuh"

extern "C" {
typedef struct {
    int32_t rows;
    int32_t cols;
    int64_t nnz;
    int64_t* rpt;
    int32_t* col;
} spnnz_gen_csr;
int spnnz_gen_rmat(int log2n, int64_t draws, double a, double b, double c, uint64_t seed, int threads,
                   spnnz_gen_csr* out);
void spnnz_gen_free(spnnz_gen_csr* m);
}

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                              \
        }                                                                              \
    } while (0)

using namespace spnnz_gpu;

__device__ __forceinline__ int4 load_cols(const int4* p, uint64_t first) {
    int4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(first));
    return v;
}

template <bool GATHER>
__global__ void __launch_bounds__(128, 10) k_pattern(const int32_t* __restrict__ col, int64_t nnz,
                                                   const uint16_t* __restrict__ deg, long long* __restrict__ out) {
    const uint64_t first = policy_evict_first(), last = policy_evict_last();
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int64_t e0 = t * 16;
    if (e0 + 16 > nnz) return;
    const int4* src = reinterpret_cast<const int4*>(col + e0);
    int c[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int4 x = load_cols(src + k, first);
        c[4 * k] = x.x;
        c[4 * k + 1] = x.y;
        c[4 * k + 2] = x.z;
        c[4 * k + 3] = x.w;
    }
    long long s = 0;
    if (GATHER) {
        int d[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) d[k] = ld_keep_u16(deg + c[k], last);
#pragma unroll
        for (int k = 0; k < 16; ++k) s += d[k];
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) s += c[k];
    }
    out[t] = s;
}

// The same gathers with each 2048-entry tile of A.col brought in by one TMA
// bulk copy (cp.async.bulk, mbarrier completion) instead of per-thread LDGs:
// does taking the column stream off the LSU path leave more of the L2->SM
// request rate to the gathers?
__global__ void __launch_bounds__(128, 10) k_pattern_tma(const int32_t* __restrict__ col, int64_t nnz,
                                                       const uint16_t* __restrict__ deg, long long* __restrict__ out) {
    __shared__ __align__(128) int s_cols[2048];
    __shared__ __align__(8) unsigned long long s_bar;
    const uint64_t first = policy_evict_first(), last = policy_evict_last();
    const int64_t tile = blockIdx.x;
    if ((tile + 1) * 2048 > nnz) return;
    const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&s_bar));
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(s_cols));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(8192) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
            "l"(col + tile * 2048), "r"(8192), "r"(bar), "l"(first)
            : "memory");
    }
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(bar)
        : "memory");
    const int i0 = threadIdx.x * 16;
    int c[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int kk = (k + threadIdx.x) & 3;  // rotated: fewer bank conflicts
        const int4 x = reinterpret_cast<const int4*>(s_cols + i0)[kk];
        c[4 * kk] = x.x;
        c[4 * kk + 1] = x.y;
        c[4 * kk + 2] = x.z;
        c[4 * kk + 3] = x.w;
    }
    int d[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) d[k] = ld_keep_u16(deg + c[k], last);
    long long s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += d[k];
    out[tile * 128 + threadIdx.x] = s;
}

// Persistent, double-buffered: each block prefetches its next tile by TMA
// while it gathers the current one.
__global__ void __launch_bounds__(128, 8) k_pattern_tma2(const int32_t* __restrict__ col, int64_t tiles,
                                                       const uint16_t* __restrict__ deg, long long* __restrict__ out) {
    __shared__ __align__(128) int s_cols[2][2048];
    __shared__ __align__(8) unsigned long long s_bar[2];
    const uint64_t first = policy_evict_first(), last = policy_evict_last();
    uint32_t bar[2], dst[2];
    for (int b = 0; b < 2; ++b) {
        bar[b] = static_cast<uint32_t>(__cvta_generic_to_shared(&s_bar[b]));
        dst[b] = static_cast<uint32_t>(__cvta_generic_to_shared(s_cols[b]));
    }
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar[b]) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const auto issue = [&](int64_t t, int b) {
        if (threadIdx.x == 0 && t < tiles) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar[b]), "r"(8192) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst[b]),
                "l"(col + t * 2048), "r"(8192), "r"(bar[b]), "l"(first)
                : "memory");
        }
    };
    int64_t t = blockIdx.x;
    issue(t, 0);
    uint32_t phase[2] = {0, 0};
    int b = 0;
    long long s = 0;
    for (; t < tiles; t += gridDim.x, b ^= 1) {
        issue(t + gridDim.x, b ^ 1);
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(bar[b]),
            "r"(phase[b])
            : "memory");
        phase[b] ^= 1;
        const int i0 = threadIdx.x * 16;
        int c[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int kk = (k + threadIdx.x) & 3;
            const int4 x = reinterpret_cast<const int4*>(s_cols[b] + i0)[kk];
            c[4 * kk] = x.x;
            c[4 * kk + 1] = x.y;
            c[4 * kk + 2] = x.z;
            c[4 * kk + 3] = x.w;
        }
        int d[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) d[k] = ld_keep_u16(deg + c[k], last);
#pragma unroll
        for (int k = 0; k < 16; ++k) s += d[k];
        __syncthreads();  // buffer b is read before it is refilled
    }
    out[blockIdx.x * 128 + threadIdx.x] = s;
}

__global__ void k_deg(const int64_t* __restrict__ rpt, int64_t k_rows, uint16_t* __restrict__ deg) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < k_rows; k += int64_t(gridDim.x) * blockDim.x) {
        const long long d = rpt[k + 1] - rpt[k];
        deg[k] = static_cast<uint16_t>(d < 0xFFFF ? d : 0xFFFF);
    }
}

int main() {
    spnnz_gen_csr a{};
    if (spnnz_gen_rmat(24, int64_t(24) << 24, 0.45, 0.22, 0.22, 5, 0, &a) != 0) {
        std::fprintf(stderr, "generator failed\n");
        return 1;
    }
    const int64_t nnz = a.nnz, m = a.rows;
    int32_t* col;
    int64_t* rpt;
    uint16_t* deg;
    long long* out;
    CK(cudaMalloc(&col, 4 * nnz));
    CK(cudaMalloc(&rpt, 8 * (m + 1)));
    CK(cudaMalloc(&deg, 2 * m));
    const int64_t threads = nnz / 16;
    CK(cudaMalloc(&out, 8 * threads));
    CK(cudaMemcpy(col, a.col, 4 * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(rpt, a.rpt, 8 * (m + 1), cudaMemcpyHostToDevice));
    k_deg<<<148 * 16, 256>>>(rpt, m, deg);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const unsigned grid = static_cast<unsigned>((threads + 127) / 128);
    const int reps = 10;
    float ms[2] = {0, 0};
    for (int g = 0; g < 2; ++g) {
        for (int r = 0; r < 3; ++r) {  // warm-up
            if (g) k_pattern<true><<<grid, 128>>>(col, nnz, deg, out);
            else k_pattern<false><<<grid, 128>>>(col, nnz, deg, out);
        }
        CK(cudaEventRecord(e0));
        for (int r = 0; r < reps; ++r) {
            if (g) k_pattern<true><<<grid, 128>>>(col, nnz, deg, out);
            else k_pattern<false><<<grid, 128>>>(col, nnz, deg, out);
        }
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms[g], e0, e1));
        ms[g] /= reps;
    }
    float mst = 0.f;
    {
        const unsigned gt = static_cast<unsigned>(nnz / 2048);
        for (int r = 0; r < 3; ++r) k_pattern_tma<<<gt, 128>>>(col, nnz, deg, out);
        CK(cudaGetLastError());
        CK(cudaEventRecord(e0));
        for (int r = 0; r < reps; ++r) k_pattern_tma<<<gt, 128>>>(col, nnz, deg, out);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&mst, e0, e1));
        mst /= reps;
    }
    float mst2[3] = {0.f, 0.f, 0.f};
    const int per_sm[3] = {4, 6, 8};
    for (int v = 0; v < 3; ++v) {
        const unsigned gt = static_cast<unsigned>(148 * per_sm[v]);
        for (int r = 0; r < 3; ++r) k_pattern_tma2<<<gt, 128>>>(col, nnz / 2048, deg, out);
        CK(cudaGetLastError());
        CK(cudaEventRecord(e0));
        for (int r = 0; r < reps; ++r) k_pattern_tma2<<<gt, 128>>>(col, nnz / 2048, deg, out);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&mst2[v], e0, e1));
        mst2[v] /= reps;
    }
    const double n = double(threads) * 16;
    std::printf("config 5 A.col: %lld nonzeros (A.col %.2f GB, degree array %.1f MB)\n", (long long)nnz,
                4.0 * nnz / 1e9, 2.0 * m / 1e6);
    std::printf("stream A.col only      : %.3f ms  %.0f GB/s\n", ms[0], 4.0 * n / (ms[0] * 1e-3) / 1e9);
    std::printf("stream + degree gather : %.3f ms  %.1f G gathers/s\n", ms[1], n / (ms[1] * 1e-3) / 1e9);
    for (int v = 0; v < 3; ++v)
        std::printf("TMA 2-stage, %d blk/SM : %.3f ms  %.1f G gathers/s\n", per_sm[v], mst2[v],
                    double(nnz / 2048) * 2048 / (mst2[v] * 1e-3) / 1e9);
    std::printf("TMA tiles + gather     : %.3f ms  %.1f G gathers/s\n", mst,
                double(nnz / 2048) * 2048 / (mst * 1e-3) / 1e9);
    spnnz_gen_free(&a);
    return 0;
}
