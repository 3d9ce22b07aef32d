// Grid-barrier / L2-broadcast microbenchmarks for the persistent kernel design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdio.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// variant 0: fence + atomicAdd + acquire spin (what pcd_wform uses)
// variant 1: red.release.gpu + acquire spin (no separate fence)
// variant 2: cooperative_groups grid.sync()
// variant 3: variant 0 + each CTA reads `nread` double2 from an L2-resident buffer per iteration
__global__ void bar_kernel(unsigned long long* ctr, int iters, int variant, const double2* buf, int nread,
                           double* sink) {
    double acc = 0.0;
    unsigned long long epoch = 0;
    for (int i = 0; i < iters; ++i) {
        if (variant == 2) {
            cg::this_grid().sync();
        } else {
            __syncthreads();
            if (threadIdx.x == 0) {
                if (variant == 1) {
                    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(ctr), "l"(1ull) : "memory");
                } else {
                    __threadfence();
                    atomicAdd(ctr, 1ull);
                }
                const unsigned long long target = (++epoch) * gridDim.x;
                while (ld_acq(ctr) < target) {
                }
            }
            __syncthreads();
        }
        if (variant == 3) {
            for (int j = threadIdx.x; j < nread; j += blockDim.x) {
                const double2 v = __ldcg(buf + j);
                acc += v.x + v.y;
            }
        }
    }
    if (acc == 12345.0) sink[0] = acc;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* ctr;
    double2* buf;
    double* sink;
    cudaMalloc(&ctr, 8);
    cudaMalloc(&buf, 16 * 60000);
    cudaMemset(buf, 0, 16 * 60000);
    cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    struct Cfg {
        int grid, threads, variant, nread;
    } cfgs[] = {{nsm, 512, 0, 0},    {nsm, 512, 1, 0},    {nsm, 512, 2, 0},     {74, 512, 0, 0},
                {32, 512, 0, 0},     {8, 512, 0, 0},      {nsm, 512, 3, 1000},  {nsm, 512, 3, 5000},
                {nsm, 512, 3, 20000}, {nsm, 1024, 0, 0},  {nsm, 128, 0, 0}};
    for (auto& c : cfgs) {
        cudaMemset(ctr, 0, 8);
        void* args[] = {&ctr, (void*)&iters, &c.variant, &buf, &c.nread, &sink};
        cudaEventRecord(e0);
        cudaError_t e = cudaLaunchCooperativeKernel((void*)bar_kernel, dim3(c.grid), dim3(c.threads), args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("grid=%3d threads=%4d variant=%d nread=%5d : %s %.3f us/barrier\n", c.grid, c.threads, c.variant,
               c.nread, e == cudaSuccess ? "ok" : cudaGetErrorString(e), ms * 1e3 / iters);
    }
    return 0;
}
