// Does a GPU-scope fence by one warp wait for other warps' outstanding global stores?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fencebench tools/fencebench.cu
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void kern(double* buf, size_t n, double* flag, int iters, int mode, unsigned long long* out) {
    const int warp = threadIdx.x >> 5;
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    if (warp == 0) {
        long long acc = 0;
        for (int i = 0; i < iters; ++i) {
            const long long t0 = clock64();
            if (threadIdx.x == 0) {
                flag[blockIdx.x * 16] = (double)i;
                if (mode & 1) __threadfence();
                else asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
            __syncwarp();
            acc += clock64() - t0;
        }
        if (threadIdx.x == 0) {
            out[blockIdx.x] = acc / iters;
            done = 1;
        }
    } else if ((mode & 2) && ((mode & 4) ? blockIdx.x != 0 : (mode & 8) ? blockIdx.x == 0 : true)) {
        // streaming stores (and loads) by the other warps until warp 0 finishes
        size_t i = (size_t)blockIdx.x * (blockDim.x - 32) + threadIdx.x - 32;
        const size_t stride = (size_t)gridDim.x * (blockDim.x - 32);
        double v = 1.0;
        volatile int* dn = (mode & 4) ? nullptr : &done;
        long long tstart = clock64();
        while (dn ? !*dn : (clock64() - tstart < 20000000)) {
            for (int k = 0; k < 16; ++k) {
                buf[i] = v;
                i += stride;
                if (i >= n) i -= n;
            }
            v += 1.0;
        }
    }
}

int main() {
    const size_t n = (size_t)1 << 28;  // 2 GB
    double *buf, *flag;
    unsigned long long* out;
    cudaMalloc(&buf, n * sizeof(double));
    cudaMalloc(&flag, 148 * 16 * sizeof(double));
    cudaMalloc(&out, 148 * sizeof(unsigned long long));
    unsigned long long h[148];
    for (int mode : {0, 2, 2 | 4, 2 | 8}) {
        kern<<<148, 512>>>(buf, n, flag, 2000, mode, out);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
        unsigned long long s = 0;
        for (int i = 0; i < 148; ++i) s += h[i];
        printf("  CTA0 only: %llu cycles\n", h[0]);
        printf("mode=%d (%s fence, %s other-warp stores): %s avg %.0f cycles per store+fence\n", mode,
               (mode & 1) ? "threadfence" : "acq_rel", (mode & 2) ? "with" : "without",
               e == cudaSuccess ? "ok" : cudaGetErrorString(e), s / 148.0);
    }
    return 0;
}
