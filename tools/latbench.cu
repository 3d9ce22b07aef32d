// Latency of a round of independent random-row loads (the stage-loop access pattern).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/latbench tools/latbench.cu
// Every CTA (148) has one warp that repeatedly issues NL independent loads, each a
// 256-byte row segment at a pseudo-random row of an S-byte array, and waits for all.
#include <cuda_runtime.h>
#include <stdio.h>

template <int NL>
__global__ void lat_kernel(const double* __restrict__ a, long long rows, int iters, int mode, double* sink,
                           unsigned long long* out) {
    unsigned long long seed = blockIdx.x * 977 + 13 + threadIdx.x / 32 * 7919;
    double acc = 0.0;
    long long t_total = 0;
    for (int it = 0; it < iters; ++it) {
        long long r[NL];
#pragma unroll
        for (int i = 0; i < NL; ++i) {
            seed = seed * 6364136223846793005ull + 1442695040888963407ull;
            r[i] = (long long)((seed >> 20) % (unsigned long long)rows);
        }
        const long long t0 = clock64();
        double v[NL];
#pragma unroll
        for (int i = 0; i < NL; ++i) {
            const double* ptr = a + r[i] * 32 + (threadIdx.x & 31);
            v[i] = (mode == 0) ? __ldg(ptr) : __ldcg(ptr);
        }
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < NL; ++i) s += v[i];
        acc += s;
        __syncwarp();
        t_total += clock64() - t0;
    }
    if (acc == 1.2345) sink[0] = acc;
    if (threadIdx.x == 0) out[blockIdx.x] = t_total / iters;
}

int main() {
    const size_t bytes = (size_t)600 << 20;
    double* a;
    double* sink;
    unsigned long long* out;
    cudaMalloc(&a, bytes);
    cudaMemset(a, 0, bytes);
    cudaMalloc(&sink, 8);
    cudaMalloc(&out, 148 * 8);
    unsigned long long h[148];
    const long long rows_all = (long long)(bytes / 256);
    for (int mode = 0; mode < 2; ++mode)
        for (long long rows : {rows_all, (long long)(32 << 20) / 256}) {
            for (int nl : {1, 10}) for (int nw : {1, 4, 16}) {
                if (nl == 1) lat_kernel<1><<<148, 32 * nw>>>(a, rows, 2000, mode, sink, out);
                else lat_kernel<10><<<148, 32 * nw>>>(a, rows, 2000, mode, sink, out);
                cudaDeviceSynchronize();
                cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
                double s = 0;
                for (int i = 0; i < 148; ++i) s += h[i];
                printf("mode=%s array=%5lld MB loads/round=%2d warps/SM=%2d : %.0f cycles per round\n", mode ? "ldcg" : "ldg ",
                       rows * 256 >> 20, nl, nw, s / 148);
            }
        }
    return 0;
}
