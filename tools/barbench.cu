// Grid-barrier variants inside the colour-chain shape (see chainbench.cu).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/barbench tools/barbench.cu
// Each phase: barrier, then every publisher thread reads two entries of the
// previous phase (L2) and writes its own entry of this phase.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_rlx(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acqrel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ int hashp(int c, int k, int p) {
    return (int)(((unsigned)c * 2654435761u + (unsigned)k * 40503u) % (unsigned)p);
}

// bar 0: __threadfence + atomicAdd + acquire poll of the counter (pcd_wform today)
// bar 1: red.release.gpu.add + acquire poll of the counter
// bar 2: per-CTA flag words (packed), st.release by thread 0; warp 0 polls all flags (relaxed) then fence
// bar 3: per-CTA flags, one 128B line each
// bar 4: two-level: 8 group counters (own lines) + red.release; warp 0 lanes poll the 8 group counters
// bar 5: like 2 but warp 0 polls with ld.acquire
__global__ void kern(int bar, int p, int w, int phases, double* buf, unsigned long long* ctr,
                     unsigned long long* flags, double* sink, int ngroups) {
    const int b = blockIdx.x, tid = threadIdx.x, nblk = gridDim.x, lane = tid & 31;
    const int c = b * w + tid;
    const bool pub = tid < w && c < p;
    double acc = 1.0;
    for (int k = 1; k < phases; ++k) {
        const unsigned long long ep = (unsigned long long)k;
        __syncthreads();
        if (bar == 0) {
            if (tid == 0) {
                __threadfence();
                atomicAdd(ctr, 1ull);
                while (ld_acq(ctr) < ep * nblk) {
                }
            }
        } else if (bar == 1) {
            if (tid == 0) {
                asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(ctr), "l"(1ull) : "memory");
                while (ld_acq(ctr) < ep * nblk) {
                }
            }
        } else if (bar == 2 || bar == 3 || bar == 5) {
            const int stride = (bar == 3) ? 16 : 1;
            if (tid == 0) st_rel(flags + (size_t)b * stride, ep);
            if (tid < 32) {
                for (int j = lane; j < nblk; j += 32) {
                    if (bar == 5) {
                        while (ld_acq(flags + (size_t)j * stride) < ep) {
                        }
                    } else {
                        while (ld_rlx(flags + (size_t)j * stride) < ep) {
                        }
                    }
                }
                __syncwarp();
                if (bar != 5) fence_acqrel();
            }
        } else if (bar == 4) {
            const int g = b % ngroups;
            const int gsize = nblk / ngroups + (g < nblk % ngroups ? 1 : 0);
            if (tid == 0)
                asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(ctr + 16 * g), "l"(1ull) : "memory");
            if (tid < 32) {
                if (lane < ngroups) {
                    const int gs = nblk / ngroups + (lane < nblk % ngroups ? 1 : 0);
                    while (ld_acq(ctr + 16 * lane) < ep * gs) {
                    }
                }
                (void)gsize;
                __syncwarp();
            }
        }
        __syncthreads();
        if (pub) {
            const double a = __ldcg(buf + (size_t)(k - 1) * p + hashp(c, k, p));
            const double bb = __ldcg(buf + (size_t)(k - 1) * p + hashp(c + 7, k, p));
            acc = a * 0.5 + bb * 0.25 + 1.0;
            buf[(size_t)k * p + c] = acc;
        }
    }
    if (acc == 12345.0) sink[0] = acc;
}

int main() {
    const int p = 5000, phases = 4000;
    double* buf;
    unsigned long long *ctr, *flags;
    double* sink;
    cudaMalloc(&buf, sizeof(double) * (size_t)p * phases);
    cudaMemset(buf, 0, sizeof(double) * (size_t)p * phases);
    cudaMalloc(&ctr, 8 * 16 * 64);
    cudaMalloc(&flags, 8 * 16 * 1024);
    cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Cfg {
        int bar, nblk, threads, ngroups;
    } cfgs[] = {{0, 148, 64, 1}, {1, 148, 64, 1}, {2, 148, 64, 1}, {3, 148, 64, 1}, {5, 148, 64, 1},
                {4, 148, 64, 8}, {4, 148, 64, 16}, {4, 148, 64, 4}, {0, 148, 512, 1}, {2, 148, 512, 1},
                {3, 148, 512, 1}};
    for (auto& cf : cfgs) {
        const int w = (p + cf.nblk - 1) / cf.nblk;
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(ctr, 0, 8 * 16 * 64);
            cudaMemset(flags, 0, 8 * 16 * 1024);
            cudaDeviceSynchronize();
            int bar = cf.bar, pp = p, ww = w, ph = phases, ng = cf.ngroups;
            void* args[] = {&bar, &pp, &ww, &ph, &buf, &ctr, &flags, &sink, &ng};
            cudaEventRecord(e0);
            cudaError_t e = cudaLaunchCooperativeKernel((void*)kern, dim3(cf.nblk), dim3(cf.threads), args, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 1)
                printf("bar=%d nblk=%3d threads=%4d groups=%2d : %s %.3f us/phase\n", cf.bar, cf.nblk, cf.threads,
                       cf.ngroups, e == cudaSuccess ? "ok" : cudaGetErrorString(e), ms * 1e3 / phases);
        }
    }
    return 0;
}
