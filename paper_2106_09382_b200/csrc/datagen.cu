// On-device synthetic data for the large configurations.
//
// The reference draws X ~ N(0, inv(Omega_true)) with a dense Cholesky of the
// truth and a dense triangular solve (datagen.py:135-154) -- O(p^3) host work
// and an n x p host->device copy (4 GB at p=50000, n=10000).  For the AR(2)
// truth (datagen.py:64-78) the Cholesky factor L is banded (two
// sub-diagonals), so each sample is one backward recurrence
//     x_i = (z_i - L[i+1,i] x_{i+1} - L[i+2,i] x_{i+2}) / L[i,i],  i = p-1 .. 0
// (L^T x = z, the system sample_mvn solves).  One thread per sample runs it
// with z from a counter-based Philox stream; the samples are written
// sample-minor (coalesced), then transposed into the n x p row-major X the
// Gram kernel takes, centred on the way (model.py:182-187).  Same
// distribution as the reference sampler, different random stream.
#include <cuda_runtime.h>
#include <curand_kernel.h>
#include <stdint.h>

namespace concord {

// XT[i][t] (p x n, row-major) = sample t, variable i.  lb: lower banded factor, lb[k*p + i] = L[i+k, i].
__global__ void ar2_sample_kernel(const double* __restrict__ lb, int p, long long n, unsigned long long seed,
                                  double* __restrict__ XT) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= n) return;
    curandStatePhilox4_32_10_t rng;
    curand_init(seed, (unsigned long long)t, 0ull, &rng);
    double x1 = 0.0, x2 = 0.0;  // x_{i+1}, x_{i+2}
    for (int i = p - 1; i >= 0; --i) {
        const double z = curand_normal_double(&rng);
        const double l1 = (i + 1 < p) ? __ldg(lb + p + i) : 0.0;
        const double l2 = (i + 2 < p) ? __ldg(lb + 2 * (long long)p + i) : 0.0;
        const double x = (z - l1 * x1 - l2 * x2) / __ldg(lb + i);
        XT[(long long)i * n + t] = x;
        x2 = x1;
        x1 = x;
    }
}

// Scale-free truth (datagen.py:99-132): a preferential-attachment TREE plus the unit diagonal,
// where every vertex v >= 1 attaches to an earlier vertex parent[v] < v.  Eliminating leaves
// first (decreasing index) factors the truth with no fill: L[v,v] = ldiag[v] and the only
// sub-diagonal entry of column v is L[parent[v], v] = lpar[v] (host: synth.tree_cholesky).
// L^T x = z is then one recurrence per sample from the root down:
//     x_v = (z_v - lpar[v] * x_parent[v]) / ldiag[v],  v = 0 .. p-1   (parent[0] = -1)
// The parent's value of the same sample is read back from XT (sample-minor, coalesced).
__global__ void tree_sample_kernel(const int* __restrict__ parent, const double* __restrict__ lpar,
                                   const double* __restrict__ ldiag, int p, long long n, unsigned long long seed,
                                   double* __restrict__ XT) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= n) return;
    curandStatePhilox4_32_10_t rng;
    curand_init(seed, (unsigned long long)t, 0ull, &rng);
    for (int v = 0; v < p; ++v) {
        const double z = curand_normal_double(&rng);
        const int u = __ldg(parent + v);
        const double xp = (u >= 0) ? XT[(long long)u * n + t] : 0.0;
        XT[(long long)v * n + t] = (z - __ldg(lpar + v) * xp) / __ldg(ldiag + v);
    }
}

// Mean over the n samples of every variable (row i of XT), two-level sum in double.
__global__ void row_mean_kernel(const double* __restrict__ XT, int p, long long n, double* __restrict__ mean) {
    __shared__ double sred[32];
    for (int i = blockIdx.x; i < p; i += gridDim.x) {
        double s = 0.0;
        for (long long t = threadIdx.x; t < n; t += blockDim.x) s += XT[(long long)i * n + t];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tot = 0.0;
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) tot += sred[k];
            mean[i] = tot / (double)n;
        }
        __syncthreads();
    }
}

// X[t][i] = XT[i][t] - mean[i]  (32 x 32 shared-memory tiles, both sides coalesced)
__global__ void transpose_center_kernel(const double* __restrict__ XT, const double* __restrict__ mean, int p,
                                        long long n, double* __restrict__ X) {
    __shared__ double tile[32][33];
    const long long t0 = (long long)blockIdx.x * 32;
    const int i0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = i0 + r;
        const long long t = t0 + threadIdx.x;
        if (i < p && t < n) tile[r][threadIdx.x] = XT[(long long)i * n + t] - mean[i];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const long long t = t0 + r;
        const int i = i0 + threadIdx.x;
        if (i < p && t < n) X[t * p + i] = tile[threadIdx.x][r];
    }
}

cudaError_t launch_ar2_sample(const double* lb, int p, long long n, unsigned long long seed, double* XT, double* mean,
                              double* X, cudaStream_t st) {
    ar2_sample_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(lb, p, n, seed, XT);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    row_mean_kernel<<<p < 148 * 8 ? p : 148 * 8, 256, 0, st>>>(XT, p, n, mean);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    transpose_center_kernel<<<dim3((unsigned)((n + 31) / 32), (unsigned)((p + 31) / 32)), dim3(32, 8), 0, st>>>(
        XT, mean, p, n, X);
    return cudaGetLastError();
}

cudaError_t launch_tree_sample(const int* parent, const double* lpar, const double* ldiag, int p, long long n,
                               unsigned long long seed, double* XT, double* mean, double* X, cudaStream_t st) {
    tree_sample_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(parent, lpar, ldiag, p, n, seed, XT);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    row_mean_kernel<<<p < 148 * 8 ? p : 148 * 8, 256, 0, st>>>(XT, p, n, mean);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    transpose_center_kernel<<<dim3((unsigned)((n + 31) / 32), (unsigned)((p + 31) / 32)), dim3(32, 8), 0, st>>>(
        XT, mean, p, n, X);
    return cudaGetLastError();
}

}  // namespace concord
