// Microbenchmarks that size the symbolic-kernel design choices on B200:
// atomic throughput (smem, DSMEM, global/L2) and random-gather throughput.
// Not part of the product; results are summarised in DESIGN.md / profiles/.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

// (1) smem atomicOr with return into a 128 KB bitmap, random bits
__global__ void k_smem_atomic(int iters, unsigned long long* out) {
    extern __shared__ uint32_t bm[];
    const int words = 32768;
    for (int i = threadIdx.x; i < words; i += blockDim.x) bm[i] = 0;
    __syncthreads();
    uint32_t s = hash32(blockIdx.x * 1024 + threadIdx.x);
    unsigned cnt = 0;
    for (int i = 0; i < iters; ++i) {
        s = hash32(s + i);
        uint32_t w = (s >> 5) & (words - 1), b = 1u << (s & 31);
        uint32_t old = atomicOr(&bm[w], b);
        cnt += !(old & b);
    }
    atomicAdd(out, cnt);
}

// (1b) smem red (no return) then popcount
__global__ void k_smem_red(int iters, unsigned long long* out) {
    extern __shared__ uint32_t bm[];
    const int words = 32768;
    for (int i = threadIdx.x; i < words; i += blockDim.x) bm[i] = 0;
    __syncthreads();
    uint32_t s = hash32(blockIdx.x * 1024 + threadIdx.x);
    for (int i = 0; i < iters; ++i) {
        s = hash32(s + i);
        uint32_t w = (s >> 5) & (words - 1), b = 1u << (s & 31);
        asm volatile("red.shared.or.b32 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(&bm[w])), "r"(b) : "memory");
    }
    __syncthreads();
    unsigned cnt = 0;
    for (int i = threadIdx.x; i < words; i += blockDim.x) cnt += __popc(bm[i]);
    atomicAdd(out, cnt);
}

// (2) DSMEM: cluster of CS CTAs, each owns 128 KB; random owner
__global__ void k_dsmem(int iters, unsigned long long* out) {
    extern __shared__ uint32_t bm[];
    cg::cluster_group cl = cg::this_cluster();
    const int words = 32768;
    for (int i = threadIdx.x; i < words; i += blockDim.x) bm[i] = 0;
    cl.sync();
    const unsigned cs = cl.num_blocks();
    uint32_t s = hash32(blockIdx.x * 1024 + threadIdx.x);
    unsigned cnt = 0;
    for (int i = 0; i < iters; ++i) {
        s = hash32(s + i);
        uint32_t w = (s >> 5) & (words - 1), b = 1u << (s & 31);
        uint32_t* remote = cl.map_shared_rank(bm, (s >> 20) % cs);
        uint32_t old = atomicOr(&remote[w], b);
        cnt += !(old & b);
    }
    cl.sync();
    atomicAdd(out, cnt);
}

// (3) global atomicOr with return into a region of `words` words
__global__ void k_global_atomic(uint32_t* bm, uint32_t words_mask, int iters, unsigned long long* out) {
    uint32_t s = hash32(blockIdx.x * 1024 + threadIdx.x);
    unsigned cnt = 0;
    for (int i = 0; i < iters; ++i) {
        s = hash32(s + i);
        uint32_t w = (s >> 5) & words_mask, b = 1u << (s & 31);
        uint32_t old = atomicOr(&bm[w], b);
        cnt += !(old & b);
    }
    atomicAdd(out, cnt);
}

// (3b) global red.or (no return)
__global__ void k_global_red(uint32_t* bm, uint32_t words_mask, int iters) {
    uint32_t s = hash32(blockIdx.x * 1024 + threadIdx.x);
    for (int i = 0; i < iters; ++i) {
        s = hash32(s + i);
        uint32_t w = (s >> 5) & words_mask, b = 1u << (s & 31);
        atomicOr(&bm[w], b);  // result unused -> RED
    }
}

// (4) random 4-byte gathers from an array of n words (independent, 8 in flight)
__global__ void k_gather32(const int32_t* __restrict__ a, uint32_t mask, int iters, unsigned long long* out) {
    uint32_t s = hash32(blockIdx.x * 1024 + threadIdx.x);
    int acc = 0;
    for (int i = 0; i < iters; i += 8) {
        int v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) { s = hash32(s + i + k); v[k] = __ldg(&a[s & mask]); }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k];
    }
    if (acc == 0x12345) atomicAdd(out, 1ull);
}

// (5) random pair gathers rpt[k], rpt[k+1] (int64) from an array of n+1
__global__ void k_gather64pair(const int64_t* __restrict__ a, uint32_t mask, int iters, unsigned long long* out) {
    uint32_t s = hash32(blockIdx.x * 1024 + threadIdx.x);
    long long acc = 0;
    for (int i = 0; i < iters; i += 8) {
        long long v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) { s = hash32(s + i + k); uint32_t j = s & mask; v[k] = __ldg(&a[j + 1]) - __ldg(&a[j]); }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k];
    }
    if (acc == 0x12345) atomicAdd(out, 1ull);
}

// (6) streaming copy int64 (for the HBM reference)
__global__ void k_copy(const int4* __restrict__ a, int4* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
    printf("device %s SMs %d L2 %d MB smemOptin %zu clock %d kHz\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin, p.clockRate);
    const int sms = p.multiProcessorCount;
    unsigned long long* d_out; CK(cudaMalloc(&d_out, 8));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    auto report = [&](const char* name, double ops) { cudaEventElapsedTime(&ms, e0, e1); printf("%-34s %8.3f ms  %8.1f Gop/s\n", name, ms, ops / ms / 1e6); };

    CK(cudaFuncSetAttribute(k_smem_atomic, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    CK(cudaFuncSetAttribute(k_smem_red, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    CK(cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    CK(cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int threads : {256, 512, 1024}) {
        int iters = 4096;
        double ops = (double)sms * threads * iters;
        k_smem_atomic<<<sms, threads, 131072>>>(16, d_out);
        cudaEventRecord(e0); k_smem_atomic<<<sms, threads, 131072>>>(iters, d_out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        char nm[64]; snprintf(nm, 64, "smem atomicOr ret (thr %d)", threads); report(nm, ops);
        cudaEventRecord(e0); k_smem_red<<<sms, threads, 131072>>>(iters, d_out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        snprintf(nm, 64, "smem red.or (thr %d)", threads); report(nm, ops);
    }
    for (int cs : {2, 4, 8, 16}) {
        int threads = 1024, iters = 2048;
        int grid = (sms / cs) * cs;
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = grid; cfg.blockDim = threads; cfg.dynamicSmemBytes = 131072;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaEventRecord(e0);
        cudaError_t err = cudaLaunchKernelEx(&cfg, k_dsmem, iters, d_out);
        cudaEventRecord(e1);
        if (err != cudaSuccess) { printf("dsmem cs=%d launch: %s\n", cs, cudaGetErrorString(err)); cudaGetLastError(); continue; }
        CK(cudaEventSynchronize(e1));
        int maxc = 0; cudaOccupancyMaxActiveClusters(&maxc, k_dsmem, &cfg);
        char nm[64]; snprintf(nm, 64, "dsmem atomicOr ret (cluster %d, act %d)", cs, maxc); report(nm, (double)grid * threads * iters);
    }
    uint32_t* d_bm; size_t big = 1ull << 30; CK(cudaMalloc(&d_bm, big)); CK(cudaMemset(d_bm, 0, big));
    for (size_t region : {2ull << 20, 16ull << 20, 64ull << 20, 1ull << 30}) {
        uint32_t mask = (uint32_t)(region / 4 - 1);
        int iters = 1024, threads = 512, grid = sms * 4;
        double ops = (double)grid * threads * iters;
        k_global_atomic<<<grid, threads>>>(d_bm, mask, 16, d_out);
        cudaEventRecord(e0); k_global_atomic<<<grid, threads>>>(d_bm, mask, iters, d_out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        char nm[64]; snprintf(nm, 64, "global atomicOr ret (%zu MB)", region >> 20); report(nm, ops);
        cudaEventRecord(e0); k_global_red<<<grid, threads>>>(d_bm, mask, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        snprintf(nm, 64, "global red.or (%zu MB)", region >> 20); report(nm, ops);
    }
    for (size_t region : {16ull << 20, 64ull << 20, 128ull << 20, 256ull << 20, 1ull << 30}) {
        int iters = 1024, threads = 512, grid = sms * 4;
        double ops = (double)grid * threads * iters;
        uint32_t mask = (uint32_t)(region / 4 - 1);
        k_gather32<<<grid, threads>>>((const int32_t*)d_bm, mask, 64, d_out);
        cudaEventRecord(e0); k_gather32<<<grid, threads>>>((const int32_t*)d_bm, mask, iters, d_out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        char nm[64]; snprintf(nm, 64, "gather int32 (%zu MB)", region >> 20); report(nm, ops);
        uint32_t mask64 = (uint32_t)(region / 8 - 2);
        mask64 = (1u << (31 - __builtin_clz(mask64))) - 1;
        cudaEventRecord(e0); k_gather64pair<<<grid, threads>>>((const int64_t*)d_bm, mask64, iters, d_out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        snprintf(nm, 64, "gather int64 pair (%zu MB)", region >> 20); report(nm, ops);
    }
    {
        size_t n = (1ull << 29) / 16;  // 512 MB each way
        int4 *a = (int4*)d_bm, *b = (int4*)((char*)d_bm + (512ull << 20));
        k_copy<<<sms * 8, 512>>>(a, b, n);
        cudaEventRecord(e0); k_copy<<<sms * 8, 512>>>(a, b, n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf("copy 512MB->512MB  %8.3f ms  %8.1f GB/s\n", ms, 1024.0 * 1.048576 / ms);
    }
    CK(cudaGetLastError());
    return 0;
}
