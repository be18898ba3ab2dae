// Does TMA gather4 beat the L1 path for random 2-byte gathers?  Measures
// random uint16 gathers from a 32 MB array (the config-5 degree array size):
// (a) plain LDG, (b) cp.async.bulk.tensor.2d ... tile::gather4 of 16-byte rows.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

__global__ void k_ldg(const uint16_t* __restrict__ a, uint32_t mask, int iters, unsigned long long* out) {
    uint32_t s = hash32(blockIdx.x * 1024 + threadIdx.x);
    unsigned acc = 0;
    for (int i = 0; i < iters; i += 8) {
        uint16_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) { s = hash32(s + i + k); v[k] = __ldg(&a[s & mask]); }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k];
    }
    if (acc == 0x12345) atomicAdd(out, 1ull);
}

// Each thread issues `per` gather4 ops per round (4 random 16-byte rows each)
// into its own smem slots; one mbarrier tracks the bytes of the round.
template <int THREADS, int PER>
__global__ void __launch_bounds__(THREADS) k_gather4(const __grid_constant__ CUtensorMap tmap,
                                                     uint32_t rows_mask, int rounds,
                                                     unsigned long long* out) {
    __shared__ __align__(128) uint8_t buf[THREADS * PER * 128];  // TMA dst: 128-byte aligned slots
    __shared__ __align__(8) uint64_t bar;
    const uint32_t bar_s = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar_s), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    uint32_t s = hash32(blockIdx.x * 4096 + threadIdx.x);
    uint32_t phase = 0;
    unsigned acc = 0;
    for (int r = 0; r < rounds; ++r) {
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar_s),
                         "r"(THREADS * PER * 64));
        __syncthreads();
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            int idx[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) { s = hash32(s + r * 131 + k * 7 + j); idx[j] = s & rows_mask; }
            const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(buf + (threadIdx.x * PER + k) * 128));
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                :: "r"(dst), "l"(&tmap), "r"(0), "r"(idx[0]), "r"(idx[1]), "r"(idx[2]), "r"(idx[3]),
                   "r"(bar_s) : "memory");
        }
        // wait for the round's bytes
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n"
            " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            " @!p bra WAIT_%=;\n}" :: "r"(bar_s), "r"(phase) : "memory");
        phase ^= 1;
        acc += buf[threadIdx.x * 128];
        __syncthreads();
    }
    if (acc == 0x12345) atomicAdd(out, 1ull);
}

// Mixed: warps [0, LDGW) gather with LDG, the rest issue gather4 ops.
template <int THREADS, int LDGW, int PER>
__global__ void __launch_bounds__(THREADS) k_mixed(const __grid_constant__ CUtensorMap tmap,
                                                   const uint16_t* __restrict__ a, uint32_t mask,
                                                   uint32_t rows_mask, int rounds, int ldg_iters,
                                                   unsigned long long* out) {
    constexpr int TMAT = THREADS - LDGW * 32;
    __shared__ __align__(128) uint8_t buf[(TMAT > 0 ? TMAT : 1) * PER * 128];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t bar_s = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar_s), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    uint32_t s = hash32(blockIdx.x * 4096 + threadIdx.x);
    unsigned acc = 0;
    if (warp < LDGW) {
        for (int i = 0; i < ldg_iters; i += 8) {
            uint16_t v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) { s = hash32(s + i + k); v[k] = __ldg(&a[s & mask]); }
#pragma unroll
            for (int k = 0; k < 8; ++k) acc += v[k];
        }
    } else {
        const int t = threadIdx.x - LDGW * 32;
        uint32_t phase = 0;
        for (int r = 0; r < rounds; ++r) {
            if (t == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar_s),
                             "r"(TMAT * PER * 64));
            asm volatile("bar.sync 1, %0;" :: "r"(TMAT));
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                int idx[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) { s = hash32(s + r * 131 + k * 7 + j); idx[j] = s & rows_mask; }
                const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(buf + (t * PER + k) * 128));
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                    :: "r"(dst), "l"(&tmap), "r"(0), "r"(idx[0]), "r"(idx[1]), "r"(idx[2]), "r"(idx[3]),
                       "r"(bar_s) : "memory");
            }
            asm volatile(
                "{\n .reg .pred p;\n WAIT_%=:\n"
                " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                " @!p bra WAIT_%=;\n}" :: "r"(bar_s), "r"(phase) : "memory");
            phase ^= 1;
            acc += buf[t * 128];
            asm volatile("bar.sync 1, %0;" :: "r"(TMAT));
        }
    }
    if (acc == 0x12345) atomicAdd(out, 1ull);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main() {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    const int sms = p.multiProcessorCount;
    const size_t elems = size_t(1) << 24;  // 16 M uint16 = 32 MB
    uint16_t* d;
    CK(cudaMalloc(&d, elems * 2));
    CK(cudaMemset(d, 1, elems * 2));
    unsigned long long* dout;
    CK(cudaMalloc(&dout, 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    {
        const int iters = 2048, threads = 512, grid = sms * 4;
        k_ldg<<<grid, threads>>>(d, elems - 1, 64, dout);
        cudaEventRecord(e0);
        k_ldg<<<grid, threads>>>(d, elems - 1, iters, dout);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf("LDG u16 random gathers:       %8.1f G/s\n", double(grid) * threads * iters / ms / 1e6);
    }
    EncodeFn encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode),
                               cudaEnableDefault, &q));
    CUtensorMap tmap;
    const cuuint64_t gdim[2] = {8, elems / 8};
    const cuuint64_t gstride[1] = {16};
    const cuuint32_t box[2] = {8, 1};
    const cuuint32_t estride[2] = {1, 1};
    CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, gdim, gstride, box, estride,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", int(r)); return 1; }
    const uint32_t rows_mask = uint32_t(elems / 8 - 1);
    auto run = [&](auto kern, int threads, int per, int blocks_per_sm) -> int {
        const int rounds = 256, grid = sms * blocks_per_sm;
        kern<<<grid, threads>>>(tmap, rows_mask, 8, dout);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        kern<<<grid, threads>>>(tmap, rows_mask, rounds, dout);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        const double g = double(grid) * threads * per * 4 * rounds;
        printf("TMA gather4 thr=%4d per=%d bps=%d: %8.1f G rows/s (%.1f GB/s of 16B rows)\n", threads,
               per, blocks_per_sm, g / ms / 1e6, g * 16 / ms / 1e6);
        return 0;
    };
    run(k_gather4<128, 2>, 128, 2, 4);
    run(k_gather4<64, 4>, 64, 4, 6);
    run(k_gather4<32, 8>, 32, 8, 6);
    run(k_gather4<256, 1>, 256, 1, 6);
    run(k_gather4<128, 1>, 128, 1, 12);
    {
        // LDG alone in the mixed kernel's shape, then LDG + TMA together
        constexpr int T = 256, LW = 6, PER = 1;
        const int grid = sms * 6, ldg_iters = 1024, rounds = 256;
        k_mixed<T, LW, PER><<<grid, T>>>(tmap, d, elems - 1, rows_mask, 0, ldg_iters, dout);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        k_mixed<T, LW, PER><<<grid, T>>>(tmap, d, elems - 1, rows_mask, 0, ldg_iters, dout);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        const double gl = double(grid) * LW * 32 * ldg_iters;
        printf("mixed, LDG only (6 warps):     %8.1f G/s  (%.3f ms)\n", gl / ms / 1e6, ms);
        const float ms_ldg = ms;
        cudaEventRecord(e0);
        k_mixed<T, LW, PER><<<grid, T>>>(tmap, d, elems - 1, rows_mask, rounds, 0, dout);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        const double gt = double(grid) * (T - LW * 32) * PER * 4 * rounds;
        printf("mixed, TMA only (2 warps):     %8.1f G/s  (%.3f ms)\n", gt / ms / 1e6, ms);
        cudaEventRecord(e0);
        k_mixed<T, LW, PER><<<grid, T>>>(tmap, d, elems - 1, rows_mask, rounds, ldg_iters, dout);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf("mixed, both:                   %8.1f G/s  (%.3f ms; LDG alone %.3f)\n",
               (gl + gt) / ms / 1e6, ms, ms_ldg);
    }
    CK(cudaGetLastError());
    return 0;
}
