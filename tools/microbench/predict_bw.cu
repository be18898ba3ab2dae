// Predict-pass bandwidth microbenchmark: the ceil-view stream (read int64
// flop, write int64 min(flop, ceil(flop / cr))) at config-5 size (2^24 rows)
// against plain copies of the same bytes, to split the pass's gap to the copy
// roofline into memory-path and FP64-division shares.  L2 flushed before
// every timed launch.  Not part of the product.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "device_common.cuh"

using namespace spnnz_gpu;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

enum Mode { kCopyStream = 0, kCopyPlain = 1, kDiv = 2, kFastDiv = 3, kMulOnly = 4, kDivZero = 5 };

template <int MODE, int U>
__global__ void __launch_bounds__(256) k_stream(const int64_t* __restrict__ in, int64_t* __restrict__ out,
                                                int64_t m, double cr) {
    const int64_t pairs = m >> 1, stride = int64_t(gridDim.x) * blockDim.x;
    const longlong2* f2 = reinterpret_cast<const longlong2*>(in);
    FastDiv fd;
    fd.init(cr);
    for (int64_t i0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i0 < pairs; i0 += U * stride) {
        longlong2 f[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * stride;
            if (MODE == kCopyPlain) f[u] = i < pairs ? f2[i] : make_longlong2(0, 0);
            else f[u] = i < pairs ? ld_stream_ll2(&f2[i]) : make_longlong2(0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * stride;
            if (i >= pairs) continue;
            longlong2 o = f[u];
            if (MODE == kDiv) {
                double q;
                o.x = ceil_view(f[u].x, cr, &q);
                o.y = ceil_view(f[u].y, cr, &q);
            } else if (MODE == kDivZero) {  // 0 / cr = +0 without the division
                double q;
                o.x = f[u].x == 0 ? 0 : ceil_view(f[u].x, cr, &q);
                o.y = f[u].y == 0 ? 0 : ceil_view(f[u].y, cr, &q);
            } else if (MODE == kFastDiv) {
                o.x = ceil_of(f[u].x, fd(static_cast<double>(f[u].x)));
                o.y = ceil_of(f[u].y, fd(static_cast<double>(f[u].y)));
            } else if (MODE == kMulOnly) {  // not exact: the cost floor of any division-free variant
                o.x = ceil_of(f[u].x, static_cast<double>(f[u].x) * fd.y);
                o.y = ceil_of(f[u].y, static_cast<double>(f[u].y) * fd.y);
            }
            if (MODE == kCopyPlain) reinterpret_cast<longlong2*>(out)[i] = o;
            else st_stream_ll2(reinterpret_cast<longlong2*>(out) + i, o);
        }
    }
}

__global__ void k_flush(int4* p, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        p[i] = make_int4(int(i), 0, 0, 0);
}

template <int MODE, int U>
float run(const int64_t* in, int64_t* out, int64_t m, int grid, int4* fl, int64_t fn) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0.f;
    const int reps = 10;
    for (int r = 0; r < reps + 2; ++r) {
        k_flush<<<1184, 256>>>(fl, fn);
        cudaEventRecord(a);
        k_stream<MODE, U><<<grid, 256>>>(in, out, m, 1.0316251415443825);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 2) tot += ms;
    }
    return tot / reps;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t m = int64_t(1) << 24;
    int64_t *in, *out;
    int4* fl;
    const int64_t fn = (int64_t(512) << 20) / 16;  // 512 MB flush buffer
    CK(cudaMalloc(&in, m * 8));
    CK(cudaMalloc(&out, m * 8));
    CK(cudaMalloc(&fl, fn * 16));
    std::vector<int64_t> h(m);
    uint64_t s = 1;
    for (int64_t i = 0; i < m; ++i) {
        s = s * 6364136223846793005ULL + 1442695040888963407ULL;
        // config-5-like profile: ~20 % empty rows, the rest spread over 1..2e5
        h[i] = ((s >> 40) % 5 == 0) ? 0 : static_cast<int64_t>((s >> 33) % 200000);
    }
    CK(cudaMemcpy(in, h.data(), m * 8, cudaMemcpyHostToDevice));
    const double gb = 2.0 * m * 8 / 1e9;
    const char* names[] = {"copy .nc/.cs", "copy plain", "ceil __ddiv_rn", "ceil FastDiv", "ceil mul (inexact)",
                           "ceil, 0 shortcut"};
    for (int per : {8, 32}) {
        const int grid = sms * per;
        float t[6];
        t[0] = run<kCopyStream, 4>(in, out, m, grid, fl, fn);
        t[1] = run<kCopyPlain, 4>(in, out, m, grid, fl, fn);
        t[2] = run<kDiv, 4>(in, out, m, grid, fl, fn);
        t[3] = run<kFastDiv, 4>(in, out, m, grid, fl, fn);
        t[4] = run<kMulOnly, 4>(in, out, m, grid, fl, fn);
        t[5] = run<kDivZero, 4>(in, out, m, grid, fl, fn);
        for (int k = 0; k < 6; ++k)
            printf("blocks/SM %2d  %-20s %8.1f us  %7.1f GB/s\n", per, names[k], t[k] * 1e3, gb / (t[k] * 1e-3));
    }
    CK(cudaGetLastError());
    return 0;
}
