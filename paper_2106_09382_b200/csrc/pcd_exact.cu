// Bit-exact direct-form sweeps: the reference's kernel protocol on the GPU.
//
// These reproduce _ckernels.pyx (cd_sweep 53-65, pcd_sweep 68-102, u2_sweep
// 105-118) bit for bit: each half sum s1 = sum_u om[r,u] t[s,u] runs
// sequentially over u = 0..p-1 with separately rounded multiply and add
// (__dmul_rn/__dadd_rn, no FMA), exactly like the reference's scalar C loop,
// and the closed forms use the same operation order (common.cuh).  They back
// the sweep-level `cuda` backend module, so the reference's own driver loop
// and tests run unchanged on the GPU.  The fast W-form fit is pcd_wform.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "pcd_wform.h"

namespace concord {

// Sequential dot exactly as the reference loop: s = ((0 + a0*b0) + a1*b1) + ...
__device__ __forceinline__ double seq_dot(const double* __restrict__ a, const double* __restrict__ b, int p) {
    double s = 0.0;
    int u = 0;
    for (; u + 4 <= p; u += 4) {
        const double x0 = a[u], x1 = a[u + 1], x2 = a[u + 2], x3 = a[u + 3];
        const double y0 = __ldg(b + u), y1 = __ldg(b + u + 1), y2 = __ldg(b + u + 2), y3 = __ldg(b + u + 3);
        s = __dadd_rn(s, __dmul_rn(x0, y0));
        s = __dadd_rn(s, __dmul_rn(x1, y1));
        s = __dadd_rn(s, __dmul_rn(x2, y2));
        s = __dadd_rn(s, __dmul_rn(x3, y3));
    }
    for (; u < p; ++u) s = __dadd_rn(s, __dmul_rn(a[u], __ldg(b + u)));
    return s;
}

__device__ __forceinline__ double pair_value(const double* om, const double* t, int p, long long r, long long s,
                                             double shrink) {
    const double s1 = seq_dot(om + r * p, t + s * p, p);
    const double s2 = seq_dot(om + s * p, t + r * p, p);
    return offdiag_from_sums(s1, s2, om[r * p + s], t[r * p + r], t[s * p + s], shrink);
}

__device__ __forceinline__ double diag_value(const double* om, const double* t, int p, long long i, double n) {
    const double a = seq_dot(om + i * p, t + i * p, p);
    return diag_from_dot(a, om[i * p + i], t[i * p + i], n);
}

// One schedule cycle: rounds separated by grid barriers, then diagonals.
__global__ void __launch_bounds__(64) pcd_sweep_exact_kernel(double* om, const double* __restrict__ t, int p,
                                                              double n, double shrink,
                                                              const long long* __restrict__ rs,
                                                              const long long* __restrict__ ss,
                                                              const long long* __restrict__ offsets, int nrounds,
                                                              unsigned long long* bar) {
    const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long gsz = (long long)gridDim.x * blockDim.x;  // even: blockDim is a multiple of 32
    unsigned long long epoch = 0;
    for (int k = 0; k < nrounds; ++k) {
        const long long lo = offsets[k], hi = offsets[k + 1];
        // Two adjacent lanes per pair: the even lane runs s1, the odd lane s2.
        for (long long base = 2 * lo; base < 2 * hi; base += gsz) {
            const long long chain = base + gtid;
            const bool valid = chain < 2 * hi;
            const long long idx = chain >> 1;
            long long r = 0, s = 0;
            double part = 0.0;
            if (valid) {
                r = rs[idx];
                s = ss[idx];
                part = (chain & 1) ? seq_dot(om + s * p, t + r * p, p) : seq_dot(om + r * p, t + s * p, p);
            }
            const double other = __shfl_xor_sync(0xffffffffu, part, 1);
            if (valid && !(chain & 1)) {
                const double v = offdiag_from_sums(part, other, om[r * p + s], t[r * p + r], t[s * p + s], shrink);
                om[r * p + s] = v;
                om[s * p + r] = v;
            }
        }
        grid_barrier(bar, (++epoch) * gridDim.x);
    }
    for (long long i = gtid; i < p; i += gsz) om[i * p + i] = diag_value(om, t, p, i, n);
}

// Serial replay with immediate writes (u2_sweep) / row-major serial CD
// (cd_sweep).  One warp: lane 0 runs s1, lane 1 runs s2 for each pair.
__global__ void serial_sweep_exact_kernel(double* om, const double* __restrict__ t, int p, double n,
                                          double shrink, const long long* __restrict__ rs,
                                          const long long* __restrict__ ss, long long npairs, int row_major) {
    const int lane = threadIdx.x;
    long long r = 0, s = 1;
    for (long long idx = 0; idx < npairs; ++idx) {
        if (!row_major) {
            r = rs[idx];
            s = ss[idx];
        }
        double part = 0.0;
        if (lane == 0) part = seq_dot(om + r * p, t + s * p, p);
        if (lane == 1) part = seq_dot(om + s * p, t + r * p, p);
        const double s2 = __shfl_sync(0xffffffffu, part, 1);
        if (lane == 0) {
            const double v = offdiag_from_sums(part, s2, om[r * p + s], t[r * p + r], t[s * p + s], shrink);
            om[r * p + s] = v;
            om[s * p + r] = v;
        }
        __syncwarp();
        if (row_major) {
            if (++s == p) {
                ++r;
                s = r + 1;
            }
        }
    }
    __syncwarp();
    // The diagonal updates read only row i and write only (i, i): independent.
    for (long long i = lane; i < p; i += 32) om[i * p + i] = diag_value(om, t, p, i, n);
}

cudaError_t launch_pcd_sweep_exact(double* om, const double* t, int p, double n, double shrink,
                                   const long long* rs, const long long* ss, const long long* offsets,
                                   int nrounds, unsigned long long* bar, cudaStream_t st) {
    int per_sm = 0, dev = 0, nsm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcd_sweep_exact_kernel, 64, 0);
    if (e != cudaSuccess) return e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    long long want = ((long long)p + 63) / 64;  // two lanes per pair of the widest round
    if (want < 1) want = 1;
    int grid = (int)(want < (long long)per_sm * nsm ? want : (long long)per_sm * nsm);
    e = cudaMemsetAsync(bar, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    void* args[] = {&om, (void*)&t, &p, &n, &shrink, (void*)&rs, (void*)&ss, (void*)&offsets, &nrounds, &bar};
    return cudaLaunchCooperativeKernel((void*)pcd_sweep_exact_kernel, dim3(grid), dim3(64), args, 0, st);
}

cudaError_t launch_u2_sweep_exact(double* om, const double* t, int p, double n, double shrink,
                                  const long long* rs, const long long* ss, long long npairs, cudaStream_t st) {
    serial_sweep_exact_kernel<<<1, 32, 0, st>>>(om, t, p, n, shrink, rs, ss, npairs, 0);
    return cudaGetLastError();
}

cudaError_t launch_cd_sweep_exact(double* om, const double* t, int p, double n, double shrink, cudaStream_t st) {
    const long long npairs = (long long)p * (p - 1) / 2;
    serial_sweep_exact_kernel<<<1, 32, 0, st>>>(om, t, p, n, shrink, nullptr, nullptr, npairs, 1);
    return cudaGetLastError();
}

}  // namespace concord
