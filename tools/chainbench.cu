// Per-phase latency of the colour chain under different inter-CTA hand-off schemes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/chainbench tools/chainbench.cu
// Each phase, every "publisher" thread (one per column, p columns over nblk CTAs)
// reads two entries of the previous phase at pseudo-random columns, combines
// them and writes its own entry for the current phase (the dependency shape of
// the CONCORD colour chain: pair (r,s) of colour k needs rows r and s of colour k-1).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double ld_relaxed(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double2 ld_relaxed2(const double2* p) {
    double2 v;
    asm volatile("ld.relaxed.gpu.global.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double ld_volatile(const double* p) {
    double v;
    asm volatile("ld.volatile.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ int hashp(int c, int k, int p) { return (int)(((unsigned)c * 2654435761u + (unsigned)k * 40503u) % (unsigned)p); }

#define SENT (-12345.678)

// variant 0: barrier (fence + atomicAdd + acquire poll same addr), then loads
// variant 1: barrier with separate release flag written by last arriver, nanosleep-free poll
// variant 2: flag-in-data (8B sentinel), no barrier
// variant 3: flag-in-data (16B double2 sentinel), no barrier
__global__ void chain_kernel(int variant, int p, int w, int phases, double* buf, double2* buf2,
                             unsigned long long* ctr, unsigned long long* rel, double* sink) {
    const int b = blockIdx.x, tid = threadIdx.x, nblk = gridDim.x;
    const int c = b * w + tid;
    const bool pub = tid < w && c < p;
    double acc = 1.0;
    unsigned long long epoch = 0;
    for (int k = 1; k < phases; ++k) {
        if (variant <= 1) {
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                unsigned long long target = (++epoch) * nblk;
                if (variant == 0) {
                    atomicAdd(ctr, 1ull);
                    while (ld_acq(ctr) < target) {
                    }
                } else {
                    unsigned long long old = atomicAdd(ctr, 1ull);
                    if (old == target - 1) {
                        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(rel), "l"(epoch) : "memory");
                    } else {
                        while (ld_acq(rel) < epoch) {
                        }
                    }
                }
            }
            __syncthreads();
            if (pub) {
                const double a = __ldcg(buf + (size_t)(k - 1) * p + hashp(c, k, p));
                const double bb = __ldcg(buf + (size_t)(k - 1) * p + hashp(c + 7, k, p));
                acc = a * 0.5 + bb * 0.25 + 1.0;
                buf[(size_t)k * p + c] = acc;
            }
        } else if (variant == 2 || variant >= 4) {
            if (pub) {
                const double* s = buf + (size_t)(k - 1) * p;
                const int i0 = hashp(c, k, p), i1 = hashp(c + 7, k, p);
                double a, bb;
                do {
                    a = ld_relaxed(s + i0);
                    bb = ld_relaxed(s + i1);
                } while (a == SENT || bb == SENT);
                acc = a * 0.5 + bb * 0.25 + 1.0;
                if (variant == 2) {
                    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(buf + (size_t)k * p + c), "d"(acc) : "memory");
                } else if (variant == 4) {
                    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(buf + (size_t)k * p + c), "d"(acc) : "memory");
                    __threadfence();
                } else if (variant == 5) {
                    asm volatile("st.release.gpu.global.f64 [%0], %1;" ::"l"(buf + (size_t)k * p + c), "d"(acc) : "memory");
                } else {
                    atomicExch((unsigned long long*)(buf + (size_t)k * p + c), (unsigned long long)__double_as_longlong(acc));
                }
            }
        } else if (variant == 3) {
            if (pub) {
                const double2* s = buf2 + (size_t)(k - 1) * p;
                const int i0 = hashp(c, k, p), i1 = hashp(c + 7, k, p);
                double2 a, bb;
                do {
                    a = ld_relaxed2(s + i0);
                    bb = ld_relaxed2(s + i1);
                } while (a.x == SENT || a.y == SENT || bb.x == SENT || bb.y == SENT);
                acc = a.x * 0.5 + bb.y * 0.25 + 1.0;
                asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1,%2};" ::"l"(buf2 + (size_t)k * p + c), "d"(acc),
                             "d"(acc + 1.0)
                             : "memory");
            }
        }
    }
    if (acc == 12345.0) sink[0] = acc;
}

// two CTAs bounce a counter through separate 128B-aligned lines; mode 0 relaxed st, 1 st.release, 2 atomicExch, 3 st+fence
__global__ void pingpong_kernel(unsigned long long* a, unsigned long long* bline, int iters, int mode) {
    if (threadIdx.x) return;
    unsigned long long* mine = blockIdx.x ? bline : a;
    unsigned long long* other = blockIdx.x ? a : bline;
    for (int i = 0; i < iters; ++i) {
        const unsigned long long want = 2ull * i + (blockIdx.x ? 1 : 0);
        if (blockIdx.x) while (ld_acq(other) < want) {}
        else if (i) while (ld_acq(other) < want - 1) {}
        const unsigned long long v = want + 1;
        if (mode == 0) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(mine), "l"(v) : "memory");
        else if (mode == 1) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(mine), "l"(v) : "memory");
        else if (mode == 2) atomicExch(mine, v);
        else { asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(mine), "l"(v) : "memory"); __threadfence(); }
    }
}

__global__ void fill_kernel(double* buf, size_t n, double v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        buf[i] = v;
}

int main() {
    const int p = 5000, phases = 2000;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* buf;
    double2* buf2;
    unsigned long long *ctr, *rel;
    double* sink;
    cudaMalloc(&buf, sizeof(double) * (size_t)p * phases);
    cudaMalloc(&buf2, sizeof(double2) * (size_t)p * phases);
    cudaMalloc(&ctr, 8);
    cudaMalloc(&rel, 8);
    cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Cfg {
        int variant, nblk, threads;
    } cfgs[] = {{0, 148, 64}, {2, 148, 64}, {4, 148, 64}, {5, 148, 64}, {6, 148, 64}, {4, 40, 128}, {6, 40, 128}};
    for (auto& cf : cfgs) {
        const int w = (p + cf.nblk - 1) / cf.nblk;
        if (w > cf.threads) continue;
        for (int rep = 0; rep < 2; ++rep) {
            fill_kernel<<<1024, 256>>>(buf, (size_t)p * phases, SENT);
            fill_kernel<<<1024, 256>>>((double*)buf2, (size_t)2 * p * phases, SENT);
            fill_kernel<<<32, 256>>>(buf, p, 1.0);
            fill_kernel<<<32, 256>>>((double*)buf2, 2 * p, 1.0);
            cudaMemset(ctr, 0, 8);
            cudaMemset(rel, 0, 8);
            cudaDeviceSynchronize();
            int variant = cf.variant, pp = p, ww = w, ph = phases;
            void* args[] = {&variant, &pp, &ww, &ph, &buf, &buf2, &ctr, &rel, &sink};
            cudaEventRecord(e0);
            cudaError_t e = cudaLaunchCooperativeKernel((void*)chain_kernel, dim3(cf.nblk), dim3(cf.threads), args, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 1)
                printf("variant=%d nblk=%3d threads=%4d w=%3d : %s %.3f us/phase\n", cf.variant, cf.nblk, cf.threads, w,
                       e == cudaSuccess ? "ok" : cudaGetErrorString(e), ms * 1e3 / phases);
        }
    }
    unsigned long long* pp;
    cudaMalloc(&pp, 4096);
    for (int mode = 0; mode < 4; ++mode) {
        for (int far = 0; far < 2; ++far) {
            cudaMemset(pp, 0, 4096);
            const int iters = 20000;
            // far=1: launch 148 CTAs but only 0 and 147 work? keep simple: 2 CTAs
            void* args[] = {&pp, far ? (void*)0 : (void*)0, (void*)&iters, &mode};
            unsigned long long* bl = pp + 64;
            void* args2[] = {&pp, &bl, (void*)&iters, &mode};
            (void)args;
            cudaEventRecord(e0);
            cudaError_t e = cudaLaunchCooperativeKernel((void*)pingpong_kernel, dim3(2), dim3(32), args2, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (!far) printf("pingpong mode=%d : %s %.3f us/one-way handoff\n", mode, e == cudaSuccess ? "ok" : cudaGetErrorString(e), ms * 1e3 / (2.0 * iters));
        }
    }
    return 0;
}
