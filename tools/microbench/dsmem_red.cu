// Throughput of shared-memory atomics on a bitmap distributed over a thread-
// block cluster (DSMEM), against local shared-memory atomics: the question
// is whether a 2^24-bit bitmap held by a 16-CTA cluster (2 MB) can replace
// the heavy-row range sort (csrc/heavy.cu) at config 5.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 dsmem_red.cu -o dsmem_red
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

// every thread ORs `ops` random bits into the cluster's bitmap (words per CTA
// = smem_words); RET: returning atomics (the count-first-set variant)
template <bool RET>
__global__ void k_red(int ops, int smem_words, unsigned long long* out) {
    extern __shared__ uint32_t bm[];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned csize = cl.num_blocks();
    for (int i = threadIdx.x; i < smem_words; i += blockDim.x) bm[i] = 0;
    cl.sync();
    uint32_t seed = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9e3779b9u;
    unsigned long long cnt = 0;
    const uint32_t bits_per_cta = uint32_t(smem_words) * 32u;
    for (int k = 0; k < ops; ++k) {
        const uint32_t h = mix(seed + k);
        const uint32_t key = h % (bits_per_cta * csize);
        const unsigned rank = key / bits_per_cta;
        const uint32_t off = key % bits_per_cta;
        uint32_t* w = cl.map_shared_rank(bm, rank) + (off >> 5);
        const uint32_t bit = 1u << (off & 31);
        if (RET)
            cnt += (atomicOr(w, bit) & bit) ? 0 : 1;
        else
            atomicOr(w, bit);
    }
    cl.sync();
    if (!RET) {
        for (int i = threadIdx.x; i < smem_words; i += blockDim.x) cnt += __popc(bm[i]);
    }
    atomicAdd(out, cnt);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int words = 32768;  // 128 KB per CTA
    const int threads = 1024, ops = 256;
    cudaFuncSetAttribute(k_red<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_red<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_red<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, words * 4);
    cudaFuncSetAttribute(k_red<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, words * 4);
    for (int ret = 0; ret < 2; ++ret) {
        for (int cs : {1, 2, 4, 8, 16}) {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = cs;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            cfg.blockDim = dim3(threads);
            cfg.dynamicSmemBytes = words * 4;
            int nclusters = 0;
            cfg.gridDim = dim3(cs);
            cudaOccupancyMaxActiveClusters(&nclusters, ret ? (void*)k_red<true> : (void*)k_red<false>, &cfg);
            const int grid = (nclusters > 0 ? nclusters : 1) * cs;
            cfg.gridDim = dim3(grid);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            for (int rep = 0; rep < 2; ++rep) {
                cudaMemset(d, 0, 8);
                cudaEventRecord(a);
                cudaError_t e = ret ? cudaLaunchKernelEx(&cfg, k_red<true>, ops, words, d)
                                    : cudaLaunchKernelEx(&cfg, k_red<false>, ops, words, d);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                if (e != cudaSuccess) {
                    std::printf("cluster %d: %s\n", cs, cudaGetErrorString(e));
                    break;
                }
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                const double nops = double(grid) * threads * ops;
                if (rep == 1)
                    std::printf("%s cluster %2d: %3d clusters (%3d CTAs) %.3f ms  %.1f G atom/s  (%.2f per SM-clk at 1.965 GHz)\n",
                                ret ? "returning " : "no-return ", cs, grid / cs, grid, ms, nops / ms / 1e6,
                                nops / (ms * 1e-3) / (nsm * 1.965e9));
            }
        }
    }
    return 0;
}
