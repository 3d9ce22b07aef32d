// T = X^T X on FP64 tensor cores (DMMA, mma.sync m8n8k4 f64), sm_100a.
//
// Replaces compute_gram (model.py:190-197: raw = X.T @ X through OpenBLAS
// DGEMM, then t = 0.5*(raw + raw.T)).  tcgen05 has no FP64 kind, so the
// reference-precision contraction uses the FP64 DMMA pipe.  Only tiles with
// bi <= bj are computed; each value is written to (i, j) and (j, i), and on a
// diagonal tile only i <= j is taken, so T is exactly symmetric by
// construction and 0.5*(raw + raw^T) is the identity on it.
//
// CTA tile 64 x 64, 4 warps (2 x 2), warp tile 32 x 32 = 4 x 4 m8n8 MMAs,
// K chunk 16 samples staged in shared memory by cp.async (2-stage ring).
// Shared row stride 68 doubles (== 4 mod 16) makes the fragment loads
// bank-conflict free.
#include <cuda_runtime.h>
#include <stdint.h>

#include "pcd_wform.h"

namespace concord {

constexpr int GB = 64;    // tile edge
constexpr int GK = 16;    // samples per stage
constexpr int GLD = 68;   // padded shared row stride (doubles)
constexpr int GTHREADS = 128;

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
    const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
    const int nbytes = valid ? 8 : 0;  // 0 -> zero fill
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem), "r"(nbytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ long long out_index(int i, int c, int p, int mode, int w) {
    if (mode == 0) return (long long)i * p + c;
    const int b = c / w;
    return (long long)b * p * w + (long long)i * w + (c - b * w);
}

__global__ void __launch_bounds__(GTHREADS) gram_f64_kernel(const double* __restrict__ X, long long n, int p,
                                                            long long ldx, double* __restrict__ out, int mode,
                                                            int w) {
    const int bi = blockIdx.y, bj = blockIdx.x;
    if (bi > bj) return;
    __shared__ __align__(16) double As[2][GK][GLD];
    __shared__ __align__(16) double Bs[2][GK][GLD];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    const int i0 = bi * GB, j0 = bj * GB;

    auto load_stage = [&](int stage, long long k0) {
        // GK x GB doubles per operand = 1024; 8 per thread.
#pragma unroll
        for (int e = 0; e < (GK * GB) / GTHREADS; ++e) {
            const int lin = e * GTHREADS + tid;
            const int kk = lin / GB, cc = lin - kk * GB;
            const long long row = k0 + kk;
            const bool rv = row < n;
            const int ci = i0 + cc, cj = j0 + cc;
            cp_async8(&As[stage][kk][cc], X + (rv ? row : 0) * ldx + (ci < p ? ci : 0), rv && ci < p);
            cp_async8(&Bs[stage][kk][cc], X + (rv ? row : 0) * ldx + (cj < p ? cj : 0), rv && cj < p);
        }
        cp_async_commit();
    };

    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    const long long nchunks = (n + GK - 1) / GK;
    load_stage(0, 0);
    for (long long ch = 0; ch < nchunks; ++ch) {
        const int st = (int)(ch & 1);
        if (ch + 1 < nchunks) {
            load_stage(st ^ 1, (ch + 1) * GK);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
#pragma unroll
        for (int ks = 0; ks < GK; ks += 4) {
            const int kr = ks + (lane & 3);
            double af[4], bf[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) af[mi] = As[st][kr][wm * 32 + mi * 8 + (lane >> 2)];
#pragma unroll
            for (int nj = 0; nj < 4; ++nj) bf[nj] = Bs[st][kr][wn * 32 + nj * 8 + (lane >> 2)];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int nj = 0; nj < 4; ++nj) dmma_8x8x4(acc[mi][nj][0], acc[mi][nj][1], af[mi], bf[nj]);
        }
        __syncthreads();
    }

#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int nj = 0; nj < 4; ++nj)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int gi = i0 + wm * 32 + mi * 8 + (lane >> 2);
                const int gj = j0 + wn * 32 + nj * 8 + 2 * (lane & 3) + h;
                if (gi >= p || gj >= p) continue;
                if (bi == bj && gi > gj) continue;
                const double v = acc[mi][nj][h];
                out[out_index(gi, gj, p, mode, w)] = v;
                out[out_index(gj, gi, p, mode, w)] = v;
            }
}

// center_columns (model.py:182-187: x - x.mean(axis=0)) in place, one thread per column.
// numpy reduces axis 0 of a C-ordered array row by row (sequential adds into the
// accumulator row), then divides by n; the same sequential __dadd_rn chain and
// __ddiv_rn give its bits exactly.  The row loads of a warp are coalesced across
// columns; eight rows are loaded ahead of the add chain.
__global__ void center_columns_kernel(double* __restrict__ X, long long n, int p, long long ldx) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= p) return;
    double s = 0.0;
    long long k = 0;
    for (; k + 8 <= n; k += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(X + (k + u) * ldx + j);
#pragma unroll
        for (int u = 0; u < 8; ++u) s = __dadd_rn(s, v[u]);
    }
    for (; k < n; ++k) s = __dadd_rn(s, __ldcg(X + k * ldx + j));
    const double mu = __ddiv_rn(s, (double)n);
    for (k = 0; k < n; ++k) X[k * ldx + j] = __dsub_rn(X[k * ldx + j], mu);
}

cudaError_t launch_center_columns(double* X, long long n, int p, long long ldx, cudaStream_t st) {
    center_columns_kernel<<<(p + 127) / 128, 128, 0, st>>>(X, n, p, ldx);
    return cudaGetLastError();
}

cudaError_t launch_gram_f64(const double* X, long long n, int p, long long ldx, double* out, int out_mode, int w,
                            cudaStream_t st) {
    const int nt = (p + GB - 1) / GB;
    gram_f64_kernel<<<dim3(nt, nt), GTHREADS, 0, st>>>(X, n, p, ldx, out, out_mode, w);
    return cudaGetLastError();
}

}  // namespace concord
