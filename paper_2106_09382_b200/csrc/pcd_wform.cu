// Persistent cooperative CONCORD-PCD fit kernel (W-form), sm_100a.
//
// Replaces the reference's per-iteration loop pcd_fit (solver.py:254-294) over
// the compiled sweep pcd_sweep (_ckernels.pyx:68-102).  Instead of the two
// length-p dot products per pair (_ckernels.pyx:33-36, 16p^3 bytes per
// sweep) it maintains W = Omega * T on the device:
//   s1 = sum_u om[r,u] t[s,u] = W[r,s],   s2 = sum_u om[s,u] t[r,u] = W[s,r]
// and after a pair changes by d applies the two row streams
//   W[r,:] += d * T[s,:],   W[s,:] += d * T[r,:]
// (diagonal i: W[i,:] += d_i * T[i,:]).  Exact zeros from the soft threshold
// make most d exactly 0, and those rows are skipped exactly.
//
// Layout in HBM: T, W and dense Omega are column-block ("slab") major.  CTA b
// owns columns [b*w, b*w+w); slab b is a p x w row-major block.  A pair's row
// update only touches a CTA's own columns, so each colour needs ONE grid
// barrier: owners publish (W[partner(c), c], Omega[partner(c), c]) for their
// columns c into a ping-pong buffer, barrier, then every CTA recomputes all
// p/2 closed forms of the colour redundantly (identical arithmetic, so
// identical results in every CTA) and applies the non-zero ones to its slab.
// The max |delta| convergence metric (solver.py:287) is therefore identical in
// every CTA and the stop test needs no extra reduction.  The diagonal phase
// (_ckernels.pyx:96-102) is one dense slab stream that also folds in the
// objective trace (model.py:210-217) as 1/2 <W, Omega>.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "pcd_wform.h"

namespace concord {

constexpr int kThreads = WFORM_THREADS;
constexpr int kCap = WFORM_LIST_CAP;  // list entries (pairs) / diag rows per chunk

__global__ void __launch_bounds__(kThreads, 1) pcd_wform_kernel(WformArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int2* L_rs = reinterpret_cast<int2*>(smem_raw);
    double* L_d = reinterpret_cast<double*>(smem_raw + kCap * sizeof(int2));
    double* D_d = reinterpret_cast<double*>(smem_raw);             // diag chunk: delta
    double* D_new = reinterpret_cast<double*>(smem_raw) + kCap;    // diag chunk: new value
    int* pubrow = reinterpret_cast<int*>(smem_raw + kCap * 16);
    __shared__ int s_cnt;
    __shared__ double s_red[5][kThreads / 32];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x;
    const int p = a.p, m = a.m, w = a.w, w2 = a.w >> 1;
    const int c0 = b * w;
    const int wl = min(w, p - c0);
    double* __restrict__ Wb = a.W + (long long)b * a.slab;
    const double* __restrict__ Tb = a.T + (long long)b * a.slab;
    double* __restrict__ Ob = a.Om + (long long)b * a.slab;
    const unsigned long long nb = gridDim.x;
    unsigned long long epoch = 0;
    unsigned g = 0;  // phase counter, selects the ping-pong publish buffer

    // Publish colour 0 of the first sweep.
    if (tid < wl) {
        const int c = c0 + tid;
        const int x = circle_partner(c, 0, m);
        if (x < p) a.pub[c] = make_double2(Wb[(long long)x * w + tid], Ob[(long long)x * w + tid]);
    }
    if (b == 0 && tid == 0) a.rec_time[0] = globaltimer_ns();

    int it = 0, converged = 0;
    double dmax_blk = 0.0;
    while (it < a.max_iter) {
        double dmax = 0.0;
        int nnz = 0;  // non-zero pair deltas seen by this thread in this sweep
        // ------------------------------------------------------ colour steps
        for (int k = 0; k < m; ++k) {
            // Next phase's publish cell for each own column; prefetch it so the
            // load overlaps the barrier wait.  Rows updated in this colour are
            // re-captured by the apply loop below.
            int xn = -1;
            double2 pre = make_double2(0.0, 0.0);
            if (tid < wl) {
                const int c = c0 + tid;
                xn = (k + 1 < m) ? circle_partner(c, k + 1, m) : c;
                if (xn < p) {
                    pre = make_double2(Wb[(long long)xn * w + tid], Ob[(long long)xn * w + tid]);
                } else {
                    xn = -1;
                }
            }
            if (tid < w) pubrow[tid] = xn;
            grid_barrier(a.bar, (++epoch) * nb);
            const double2* __restrict__ pb = a.pub + (size_t)(g & 1) * p;
            double2* __restrict__ pn = a.pub + (size_t)((g + 1) & 1) * p;

            for (int q0 = 0; q0 < a.half; q0 += kCap) {
                if (tid == 0) s_cnt = 0;
                __syncthreads();
                const int qend = min(q0 + kCap, a.half);
                for (int base = q0; base < qend; base += kThreads) {
                    const int q = base + tid;
                    int r = 0, s = 0;
                    double d = 0.0;
                    if (q < qend) {
                        circle_pair(k, q, m, r, s);
                        if (s < p) {
                            const double2 vr = ldcg2(pb + r);  // (W[s,r], Om[s,r])
                            const double2 vs = ldcg2(pb + s);  // (W[r,s], Om[r,s])
                            const double trr = __ldg(a.tdiag + r), tss = __ldg(a.tdiag + s);
                            const double om = vs.y;
                            const double nv = offdiag_from_sums(vs.x, vr.x, om, trr, tss, a.shrink);
                            d = __dsub_rn(nv, om);
                            if (d != 0.0) {
                                dmax = fmax(dmax, fabs(d));
                                ++nnz;
                                if ((unsigned)(s - c0) < (unsigned)wl) Ob[(long long)r * w + (s - c0)] = nv;
                                if ((unsigned)(r - c0) < (unsigned)wl) Ob[(long long)s * w + (r - c0)] = nv;
                            }
                        }
                    }
                    const unsigned mask = __ballot_sync(0xffffffffu, d != 0.0);
                    if (mask) {
                        int basepos = 0;
                        if (lane == 0) basepos = atomicAdd(&s_cnt, __popc(mask));
                        basepos = __shfl_sync(0xffffffffu, basepos, 0);
                        if (d != 0.0) {
                            const int slot = basepos + __popc(mask & ((1u << lane) - 1u));
                            L_rs[slot] = make_int2(r, s);
                            L_d[slot] = d;
                        }
                    }
                }
                if (q0 == 0 && xn >= 0) pn[c0 + tid] = pre;
                __syncthreads();
                const int cnt = s_cnt;
                const int per = 2 * w2;
                const int items = cnt * per;
                for (int idx = tid; idx < items; idx += kThreads) {
                    const int e = idx / per;
                    const int rem = idx - e * per;
                    const int h = rem >= w2;
                    const int j2 = rem - h * w2;
                    const int2 rs = L_rs[e];
                    const double d = L_d[e];
                    const int dst = h ? rs.y : rs.x;
                    const int src = h ? rs.x : rs.y;
                    double2* wp = reinterpret_cast<double2*>(Wb + (long long)dst * w) + j2;
                    const double2 tv = __ldg(reinterpret_cast<const double2*>(Tb + (long long)src * w) + j2);
                    double2 wv = *wp;
                    wv.x = fma(d, tv.x, wv.x);
                    wv.y = fma(d, tv.y, wv.y);
                    *wp = wv;
                    const int j = 2 * j2;
                    if (pubrow[j] == dst) pn[c0 + j].x = wv.x;
                    if (pubrow[j + 1] == dst) pn[c0 + j + 1].x = wv.y;
                }
                __syncthreads();
            }
            ++g;
        }

        // ------------------------------------------------------ diagonal step
        int x0 = -1;
        double pre_om = 0.0;
        if (tid < wl) {
            const int c = c0 + tid;
            x0 = circle_partner(c, 0, m);
            if (x0 < p) pre_om = Ob[(long long)x0 * w + tid];
            else x0 = -1;
        }
        grid_barrier(a.bar, (++epoch) * nb);
        if (tid < w) pubrow[tid] = x0;
        const double2* __restrict__ pb = a.pub + (size_t)(g & 1) * p;
        double2* __restrict__ pn = a.pub + (size_t)((g + 1) & 1) * p;
        if (x0 >= 0) pn[c0 + tid].y = pre_om;  // .x is captured by the dense pass
        double q_acc = 0.0, pen_acc = 0.0, log_acc = 0.0;
        for (int i0 = 0; i0 < p; i0 += kCap) {
            const int iend = min(i0 + kCap, p);
            __syncthreads();
            for (int i = i0 + tid; i < iend; i += kThreads) {
                const double2 v = ldcg2(pb + i);  // (W[i,i], Om[i,i])
                const double tii = __ldg(a.tdiag + i);
                const double nv = diag_from_dot(v.x, v.y, tii, a.n);
                const double d = __dsub_rn(nv, v.y);
                dmax = fmax(dmax, fabs(d));
                D_d[i - i0] = d;
                D_new[i - i0] = nv;
            }
            __syncthreads();
            const int items = (iend - i0) * w2;
            for (int idx = tid; idx < items; idx += kThreads) {
                const int ii = idx / w2;
                const int j2 = idx - ii * w2;
                const int i = i0 + ii;
                const double d = D_d[ii];
                double2* wp = reinterpret_cast<double2*>(Wb + (long long)i * w) + j2;
                double2 wv = *wp;
                if (d != 0.0) {
                    const double2 tv = __ldg(reinterpret_cast<const double2*>(Tb + (long long)i * w) + j2);
                    wv.x = fma(d, tv.x, wv.x);
                    wv.y = fma(d, tv.y, wv.y);
                    *wp = wv;
                }
                const int j = 2 * j2;
                const int cj = c0 + j;
                if (pubrow[j] == i) pn[cj].x = wv.x;
                if (pubrow[j + 1] == i) pn[cj + 1].x = wv.y;
                const bool dg0 = (cj == i), dg1 = (cj + 1 == i);
                if (a.want_trace) {
                    double2* op = reinterpret_cast<double2*>(Ob + (long long)i * w) + j2;
                    double2 ov = *op;
                    if (dg0 | dg1) {
                        if (dg0) ov.x = D_new[ii];
                        if (dg1) ov.y = D_new[ii];
                        *op = ov;
                        log_acc += log(D_new[ii]);
                    }
                    q_acc = fma(wv.x, ov.x, q_acc);
                    q_acc = fma(wv.y, ov.y, q_acc);
                    if (i < cj) pen_acc += fabs(ov.x);
                    if (i < cj + 1) pen_acc += fabs(ov.y);
                } else if (dg0 | dg1) {
                    Ob[(long long)i * w + (dg0 ? j : j + 1)] = D_new[ii];
                }
            }
        }
        ++g;
        ++it;

        // ------------------------------------------------- block reductions
        dmax = warp_max(dmax);
        q_acc = warp_sum(q_acc);
        pen_acc = warp_sum(pen_acc);
        log_acc = warp_sum(log_acc);
        const double nnz_w = warp_sum((double)nnz);
        if (lane == 0) {
            s_red[0][warp] = dmax;
            s_red[1][warp] = q_acc;
            s_red[2][warp] = pen_acc;
            s_red[3][warp] = log_acc;
            s_red[4][warp] = nnz_w;
        }
        __syncthreads();
        if (warp == 0) {
            double v0 = s_red[0][lane], v1 = s_red[1][lane], v2 = s_red[2][lane], v3 = s_red[3][lane];
            const double v4 = warp_sum(s_red[4][lane]);
            v0 = warp_max(v0);
            v1 = warp_sum(v1);
            v2 = warp_sum(v2);
            v3 = warp_sum(v3);
            if (lane == 0) {
                s_red[0][0] = v0;
                if (a.want_trace) {
                    double* ro = a.rec_obj + ((size_t)(it - 1) * gridDim.x + b) * 3;
                    ro[0] = v1;
                    ro[1] = v2;
                    ro[2] = v3;
                }
                if (b == 0) {
                    a.rec_delta[it - 1] = v0;
                    a.rec_nnz[it - 1] = (long long)v4;
                    a.rec_time[it] = globaltimer_ns();
                }
            }
        }
        __syncthreads();
        dmax_blk = s_red[0][0];
        __syncthreads();
        if (dmax_blk < a.delta_tol) {
            converged = 1;
            break;
        }
    }
    if (b == 0 && tid == 0) {
        a.status[0] = it;
        a.status[1] = converged;
    }
}

// --------------------------------------------------------------- layout kernels
// Row-major p x p (leading dim ld) -> slab-major (zero padding).
__global__ void pack_slabs_kernel(const double* __restrict__ src, long long ld, double* __restrict__ dst,
                                  int p, int w, int nblk) {
    const long long total = (long long)nblk * p * w;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long b = e / ((long long)p * w);
        const long long rem = e - b * p * w;
        const int i = (int)(rem / w);
        const int j = (int)(rem - (long long)i * w);
        const long long c = b * w + j;
        dst[e] = (c < p) ? src[(long long)i * ld + c] : 0.0;
    }
}

// Slab-major -> row-major p x p.
__global__ void unpack_slabs_kernel(const double* __restrict__ src, double* __restrict__ dst, int p, int w) {
    const long long total = (long long)p * p;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e / p);
        const int c = (int)(e - (long long)i * p);
        const int b = c / w;
        dst[e] = src[(long long)b * p * w + (long long)i * w + (c - b * w)];
    }
}

__global__ void slab_diag_kernel(const double* __restrict__ slab, double* __restrict__ diag, int p, int w) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p; i += gridDim.x * blockDim.x) {
        const int b = i / w;
        diag[i] = slab[(long long)b * p * w + (long long)i * w + (i - b * w)];
    }
}

__global__ void slab_set_identity_kernel(double* __restrict__ slab, int p, int w) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p; i += gridDim.x * blockDim.x) {
        const int b = i / w;
        slab[(long long)b * p * w + (long long)i * w + (i - b * w)] = 1.0;
    }
}

// Count exact non-zeros of the strict upper triangle (model.py:249-253).
__global__ void slab_edge_count_kernel(const double* __restrict__ slab, int p, int w, int nblk,
                                       unsigned long long* __restrict__ out) {
    unsigned long long local = 0;
    const long long total = (long long)nblk * p * w;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long b = e / ((long long)p * w);
        const long long rem = e - b * p * w;
        const int i = (int)(rem / w);
        const long long c = b * w + (rem - (long long)i * w);
        if (c < p && i < c && slab[e] != 0.0) ++local;
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(out, local);
}

// W (slab) = Omega_init * T for a warm start, from a CSR copy of Omega_init.
// Row i of W is sum_k om[i,k] T[k,:]; each block streams its own slab.
__global__ void wform_init_csr_kernel(const int* __restrict__ rowptr, const int* __restrict__ colidx,
                                      const double* __restrict__ vals, const double* __restrict__ Tslab,
                                      double* __restrict__ Wslab, int p, int w) {
    const int b = blockIdx.y;
    const double* Tb = Tslab + (long long)b * p * w;
    double* Wb = Wslab + (long long)b * p * w;
    const int w2 = w >> 1;
    const long long items = (long long)p * w2;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < items;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / w2);
        const int j2 = (int)(idx - (long long)i * w2);
        double2 acc = make_double2(0.0, 0.0);
        for (int e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            const double v = vals[e];
            const double2 tv = __ldg(reinterpret_cast<const double2*>(Tb + (long long)colidx[e] * w) + j2);
            acc.x = fma(v, tv.x, acc.x);
            acc.y = fma(v, tv.y, acc.y);
        }
        reinterpret_cast<double2*>(Wb + (long long)i * w)[j2] = acc;
    }
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_pcd_wform(const WformArgs& args, int nblk, cudaStream_t st) {
    const size_t smem = wform_smem_bytes(args.w);
    cudaError_t e = cudaFuncSetAttribute(pcd_wform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    WformArgs copy = args;
    void* kargs[] = {&copy};
    return cudaLaunchCooperativeKernel((void*)pcd_wform_kernel, dim3(nblk), dim3(kThreads), kargs, smem, st);
}

cudaError_t wform_max_blocks(int w, int* max_blocks) {
    const size_t smem = wform_smem_bytes(w);
    cudaError_t e = cudaFuncSetAttribute(pcd_wform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcd_wform_kernel, kThreads, smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    *max_blocks = per_sm * nsm;
    return cudaSuccess;
}

static int grid_for(long long total) {
    long long g = (total + 255) / 256;
    if (g > 148LL * 16) g = 148LL * 16;
    if (g < 1) g = 1;
    return (int)g;
}

cudaError_t launch_pack_slabs(const double* src, long long ld, double* dst, int p, int w, int nblk,
                              cudaStream_t st) {
    pack_slabs_kernel<<<grid_for((long long)nblk * p * w), 256, 0, st>>>(src, ld, dst, p, w, nblk);
    return cudaGetLastError();
}

cudaError_t launch_unpack_slabs(const double* src, double* dst, int p, int w, cudaStream_t st) {
    unpack_slabs_kernel<<<grid_for((long long)p * p), 256, 0, st>>>(src, dst, p, w);
    return cudaGetLastError();
}

cudaError_t launch_slab_diag(const double* slab, double* diag, int p, int w, cudaStream_t st) {
    slab_diag_kernel<<<grid_for(p), 256, 0, st>>>(slab, diag, p, w);
    return cudaGetLastError();
}

cudaError_t launch_slab_identity(double* slab, int p, int w, int nblk, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(slab, 0, sizeof(double) * (size_t)nblk * p * w, st);
    if (e != cudaSuccess) return e;
    slab_set_identity_kernel<<<grid_for(p), 256, 0, st>>>(slab, p, w);
    return cudaGetLastError();
}

cudaError_t launch_slab_edge_count(const double* slab, int p, int w, int nblk, unsigned long long* out,
                                   cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    slab_edge_count_kernel<<<grid_for((long long)nblk * p * w), 256, 0, st>>>(slab, p, w, nblk, out);
    return cudaGetLastError();
}

cudaError_t launch_wform_init_csr(const int* rowptr, const int* colidx, const double* vals, const double* Tslab,
                                  double* Wslab, int p, int w, int nblk, cudaStream_t st) {
    long long items = (long long)p * (w >> 1);
    int gx = (int)((items + 255) / 256);
    if (gx > 64) gx = 64;
    wform_init_csr_kernel<<<dim3(gx, nblk), 256, 0, st>>>(rowptr, colidx, vals, Tslab, Wslab, p, w);
    return cudaGetLastError();
}

}  // namespace concord
