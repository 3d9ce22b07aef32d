// Random-row stream ceiling: how many bytes/s can 148 SMs move for the apply warps' access
// pattern W[dst, cols] = fma(d, T[src, cols], W[dst, cols]) with random dst/src rows?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/rowbench tools/rowbench.cu
// Unlike bulkbench.cu the per-item work is the kernel's: entries in shared memory, division-free
// cursors, a per-thread cp.async ring S deep.  Layouts:
//   slab     -- CTA b owns a contiguous p x w block (pcd_qblock.cu), rows of w doubles
//   rowmajor -- p x (nsm*w) row-major, CTA b owns columns [b*w, b*w+w): all CTAs reading the
//               same row at about the same time touch one contiguous DRAM region
// Every CTA applies the same entry list (like the real kernel: every CTA applies every pair
// to its own columns); one __syncthreads per pass of `nh` half-entries.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

constexpr int kThreads = 320;  // the blocked kernel's apply warps (10)

extern __shared__ __align__(16) unsigned char smem[];

template <int S>
__global__ void __launch_bounds__(kThreads, 1)
    rows_kernel(double* W, const double* T, const int2* ent, const double* dd, int w, int nh, int passes,
                long long slab, int rowmajor) {
    const int tid = threadIdx.x;
    double* __restrict__ Wb = W + (rowmajor ? (long long)blockIdx.x * w : (long long)blockIdx.x * slab);
    const double* __restrict__ Tb = T + (rowmajor ? (long long)blockIdx.x * w : (long long)blockIdx.x * slab);
    const int w2 = w / 2;
    const long long ld2 = rowmajor ? (long long)gridDim.x * w / 2 : w2;
    int2* Ls = reinterpret_cast<int2*>(smem);
    double* Ld = reinterpret_cast<double*>(smem + 8 * nh);
    double2* ring = reinterpret_cast<double2*>(smem + 16 * nh);
    for (int ps = 0; ps < passes; ++ps) {
        for (int i = tid; i < nh; i += kThreads) {
            Ls[i] = ent[(size_t)ps * nh + i];
            Ld[i] = dd[(size_t)ps * nh + i];
        }
        __syncthreads();
        const int items = nh * w2;
        const int nmine = items > tid ? (items - tid + kThreads - 1) / kThreads : 0;
        const int dq = kThreads / w2, dr = kThreads - dq * w2;
        int qi = tid / w2, ri = tid - qi * w2, qc = qi, rc = ri;
        int si = 0, sc = 0;
        auto issue = [&]() {
            const int2 rs = Ls[qi];
            double2* slot = ring + (size_t)(si * 2) * kThreads + tid;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(slot)),
                         "l"(reinterpret_cast<const double2*>(Wb) + rs.x * ld2 + ri)
                         : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             (unsigned)__cvta_generic_to_shared(slot + kThreads)),
                         "l"(reinterpret_cast<const double2*>(Tb) + rs.y * ld2 + ri)
                         : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
            si = (si + 1 == S) ? 0 : si + 1;
            qi += dq;
            ri += dr;
            if (ri >= w2) {
                ri -= w2;
                ++qi;
            }
        };
        int ni = min(nmine, S - 1);
        for (int i = 0; i < ni; ++i) issue();
        for (int j = 0; j < nmine; ++j) {
            if (ni < nmine) {
                issue();
                ++ni;
                asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            const int2 rs = Ls[qc];
            const double2* slot = ring + (size_t)(sc * 2) * kThreads + tid;
            double2 wv = slot[0];
            const double2 tv = slot[kThreads];
            const double d = Ld[qc];
            wv.x = fma(d, tv.x, wv.x);
            wv.y = fma(d, tv.y, wv.y);
            reinterpret_cast<double2*>(Wb)[rs.x * ld2 + rc] = wv;
            sc = (sc + 1 == S) ? 0 : sc + 1;
            qc += dq;
            rc += dr;
            if (rc >= w2) {
                rc -= w2;
                ++qc;
            }
        }
        __syncthreads();
    }
}

template <int S>
float run(int nsm, int w, int nh, int passes, int rowmajor, double* W, double* T, int2* ent, double* dd,
          long long slab) {
    const size_t sm = (size_t)16 * nh + (size_t)S * 2 * kThreads * 16;
    cudaFuncSetAttribute(rows_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    rows_kernel<S><<<nsm, kThreads, sm>>>(W, T, ent, dd, w, nh, passes, slab, rowmajor);
    cudaEventRecord(e0);
    rows_kernel<S><<<nsm, kThreads, sm>>>(W, T, ent, dd, w, nh, passes, slab, rowmajor);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
        exit(1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    const int p = 5000, passes = 100;
    struct Cfg {
        int nsm, w, nh;
    } cfgs[] = {{148, 34, 484}, {148, 34, 1936}, {148, 36, 1936}, {148, 68, 1936}, {74, 68, 1936},
                {66, 76, 484},  {66, 76, 1936},  {41, 122, 1936}, {110, 46, 1936}};
    for (auto cf : cfgs) {
        const int nsm = cf.nsm, w = cf.w, nh = cf.nh;
        const long long slab = (long long)p * w;
        double *W, *T, *dd;
        int2* ent;
        cudaMalloc(&W, slab * nsm * 8);
        cudaMalloc(&T, slab * nsm * 8);
        cudaMemset(W, 0, slab * nsm * 8);
        cudaMemset(T, 0, slab * nsm * 8);
        cudaMalloc(&ent, sizeof(int2) * nh * passes);
        cudaMalloc(&dd, sizeof(double) * nh * passes);
        int2* he = (int2*)malloc(sizeof(int2) * nh * passes);
        double* hd = (double*)malloc(sizeof(double) * nh * passes);
        int* perm = (int*)malloc(sizeof(int) * p);
        srand(1);
        for (int ps = 0; ps < passes; ++ps) {
            for (int i = 0; i < p; ++i) perm[i] = i;
            for (int i = 0; i < nh; ++i) {
                const int j = i + rand() % (p - i);
                const int t = perm[i];
                perm[i] = perm[j];
                perm[j] = t;
                he[ps * nh + i] = make_int2(perm[i], rand() % p);
                hd[ps * nh + i] = 1e-3;
            }
        }
        cudaMemcpy(ent, he, sizeof(int2) * nh * passes, cudaMemcpyHostToDevice);
        cudaMemcpy(dd, hd, sizeof(double) * nh * passes, cudaMemcpyHostToDevice);
        const double bytes = 24.0 * w * (double)nh * passes * nsm;
        for (int rm = 0; rm < 2; ++rm) {
            float t4 = run<4>(nsm, w, nh, passes, rm, W, T, ent, dd, slab);
            float t6 = run<6>(nsm, w, nh, passes, rm, W, T, ent, dd, slab);
            float t10 = run<10>(nsm, w, nh, passes, rm, W, T, ent, dd, slab);
            float t16 = run<16>(nsm, w, nh, passes, rm, W, T, ent, dd, slab);
            printf("nsm=%3d w=%3d nh=%4d %s  GB/s device (per SM) S=4: %6.0f (%5.1f)  S=6: %6.0f (%5.1f)  "
                   "S=10: %6.0f (%5.1f)  S=16: %6.0f (%5.1f)\n",
                   nsm, w, nh, rm ? "rowmajor" : "slab    ", bytes / t4 / 1e6, bytes / t4 / 1e6 / nsm,
                   bytes / t6 / 1e6, bytes / t6 / 1e6 / nsm, bytes / t10 / 1e6, bytes / t10 / 1e6 / nsm,
                   bytes / t16 / 1e6, bytes / t16 / 1e6 / nsm);
        }
        cudaFree(W);
        cudaFree(T);
        cudaFree(ent);
        cudaFree(dd);
        free(he);
        free(hd);
        free(perm);
    }
    return 0;
}
