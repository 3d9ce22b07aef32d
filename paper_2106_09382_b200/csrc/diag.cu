// Device diagnostics on the slab-resident estimate.
//
//  * check_optimality (model.py:256-289): with M = Omega*T -- which the solver
//    already holds as W -- the stationarity violation of every coordinate is
//      diagonal  | M_ii - n / omega_ii |
//      omega_rs != 0:  | M_rs + M_sr + n*lam*sign(omega_rs) |
//      omega_rs == 0:  max(|M_rs + M_sr| - n*lam, 0)
//    reduced to the worst value and its coordinate.  One pass over the upper
//    triangle; M_sr is read from the other column's slab.
//  * estimate triplets (fileio.py:87-95): the upper-triangle entries the
//    reference's write_estimate stores (every diagonal, every exact non-zero
//    with i < j) compacted on the device in (i, j) order.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "pcd_wform.h"

namespace concord {

__device__ __forceinline__ double slab_at(const double* slab, int w, long long ss, long long rs, int i, int j) {
    const int b = j / w;
    return slab[(long long)b * ss + (long long)i * rs + (j - b * w)];
}

// Per-thread worst (value, flat index) over the upper triangle, reduced per block.
__global__ void optimality_kernel(const double* __restrict__ W, const double* __restrict__ Om, int p, int w,
                                  long long ss, long long rs,
                                  double n, double weight, double* __restrict__ blk_val,
                                  long long* __restrict__ blk_idx) {
    double best = -1.0;
    long long bidx = 0;
    const long long total = (long long)p * p;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e / p), j = (int)(e - (long long)i * p);
        if (j < i) continue;
        const double om = slab_at(Om, w, ss, rs, i, j);
        double v;
        if (i == j) {
            v = fabs(slab_at(W, w, ss, rs, i, i) - n / om);
        } else {
            const double g = slab_at(W, w, ss, rs, i, j) + slab_at(W, w, ss, rs, j, i);
            v = (om != 0.0) ? fabs(g + weight * (om > 0.0 ? 1.0 : -1.0)) : fmax(fabs(g) - weight, 0.0);
        }
        if (v > best || (v == best && e < bidx)) {
            best = v;
            bidx = e;
        }
    }
    __shared__ double sv[32];
    __shared__ long long si[32];
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, bidx, o);
        if (ov > best || (ov == best && oi < bidx)) {
            best = ov;
            bidx = oi;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        sv[warp] = best;
        si[warp] = bidx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        best = sv[0];
        bidx = si[0];
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
            if (sv[k] > best || (sv[k] == best && si[k] < bidx)) {
                best = sv[k];
                bidx = si[k];
            }
        blk_val[blockIdx.x] = best;
        blk_idx[blockIdx.x] = bidx;
    }
}

// Entries row i stores: j = i, and j > i with omega_ij != 0.
__global__ void triplet_count_kernel(const double* __restrict__ Om, int p, int w, long long ss, long long rs,
                                     int* __restrict__ rowcnt) {
    for (int i = blockIdx.x; i < p; i += gridDim.x) {
        int c = 0;
        for (int j = i + 1 + threadIdx.x; j < p; j += blockDim.x) c += slab_at(Om, w, ss, rs, i, j) != 0.0;
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        __shared__ int sc[32];
        if ((threadIdx.x & 31) == 0) sc[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 1;  // the diagonal
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sc[k];
            rowcnt[i] = t;
        }
        __syncthreads();
    }
}

// Row i writes its entries in ascending j at rowoff[i] (exclusive scan of rowcnt).
__global__ void triplet_write_kernel(const double* __restrict__ Om, int p, int w, long long ss, long long rs,
                                     const long long* __restrict__ rowoff,
                                     int* __restrict__ ti, int* __restrict__ tj, double* __restrict__ tv) {
    __shared__ int s_base;
    __shared__ int sc[32];
    for (int i = blockIdx.x; i < p; i += gridDim.x) {
        long long at = rowoff[i];
        if (threadIdx.x == 0) {
            ti[at] = i;
            tj[at] = i;
            tv[at] = slab_at(Om, w, ss, rs, i, i);
            s_base = 0;
        }
        ++at;
        __syncthreads();
        for (int j0 = i + 1; j0 < p; j0 += blockDim.x) {
            const int j = j0 + threadIdx.x;
            const double v = (j < p) ? slab_at(Om, w, ss, rs, i, j) : 0.0;
            const bool nz = v != 0.0;
            const unsigned mask = __ballot_sync(0xffffffffu, nz);
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
            if (lane == 0) sc[warp] = __popc(mask);
            __syncthreads();
            int before = 0, total = 0;
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
                if (k < warp) before += sc[k];
                total += sc[k];
            }
            if (nz) {
                const long long pos = at + s_base + before + __popc(mask & ((1u << lane) - 1u));
                ti[pos] = i;
                tj[pos] = j;
                tv[pos] = v;
            }
            __syncthreads();
            if (threadIdx.x == 0) s_base += total;
            __syncthreads();
        }
    }
}

cudaError_t launch_optimality(const double* W, const double* Om, int p, int w, long long ss, long long rs, double n,
                              double weight,
                              double* blk_val, long long* blk_idx, int nblocks, cudaStream_t st) {
    optimality_kernel<<<nblocks, 256, 0, st>>>(W, Om, p, w, ss, rs, n, weight, blk_val, blk_idx);
    return cudaGetLastError();
}

cudaError_t launch_triplet_count(const double* Om, int p, int w, long long ss, long long rs, int* rowcnt,
                                 cudaStream_t st) {
    triplet_count_kernel<<<p < 148 * 8 ? p : 148 * 8, 256, 0, st>>>(Om, p, w, ss, rs, rowcnt);
    return cudaGetLastError();
}

cudaError_t launch_triplet_write(const double* Om, int p, int w, long long ss, long long rs, const long long* rowoff,
                                 int* ti, int* tj,
                                 double* tv, cudaStream_t st) {
    triplet_write_kernel<<<p < 148 * 8 ? p : 148 * 8, 256, 0, st>>>(Om, p, w, ss, rs, rowoff, ti, tj, tv);
    return cudaGetLastError();
}

}  // namespace concord
