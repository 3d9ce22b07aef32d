// Row-stream microbenchmark: the apply warps' W[dst, slab] += d * T[src, slab] streams.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/bulkbench tools/bulkbench.cu
//   tools/bulkbench [nsm]
// Every CTA owns a p x w row-major slab of W and T (like pcd_qblock.cu) and runs `passes`
// passes; a pass applies `nh` half-entries (dst, src, d) with distinct dst rows, like one
// colour phase at lambda=0.1 (p=5000: ~242 non-zero pairs -> 484 half-entries per CTA).
// Variants (12 apply warps, 384 threads):
//   0  per-thread cp.async ring of S 32-byte items (the round-1 kernel's apply_rows_async)
//   1  per-warp bulk ring: lane 0 issues cp.async.bulk of the W and T rows into a slot,
//      mbarrier complete_tx; the warp waits, FMAs, stores W with st.global
//   2  as 1, plus fence.proxy.async.global by every lane after its stores of each slot
//   3  as 1, T rows only by bulk copy; W by per-lane ld.global issued one slot ahead
// Reports algorithmic GB/s (24 w bytes per half-entry) per SM and for the device.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

constexpr int kThreads = 384;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred P1;\n LAB_WAIT:\n"
        " mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra LAB_WAIT;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

extern __shared__ __align__(128) unsigned char smem[];

struct Args {
    double* W;
    const double* T;
    const int2* ent;  // [passes][nh] (dst, src) per CTA (same lists for every CTA)
    const double* dd;
    int p, w, nh, passes, S, Rw, variant;
    long long slab;
    int rowmajor;  // 1: W/T are p x (nsm*w) row-major (CTA b owns columns [b*w, b*w+w)); 0: slabs
};

__global__ void __launch_bounds__(kThreads, 1) rows_kernel(Args a) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* __restrict__ Wb = a.W + (a.rowmajor ? (long long)blockIdx.x * a.w : (long long)blockIdx.x * a.slab);
    const double* __restrict__ Tb = a.T + (a.rowmajor ? (long long)blockIdx.x * a.w : (long long)blockIdx.x * a.slab);
    const int w = a.w, w2 = w / 2;
    const int ld2 = a.rowmajor ? (gridDim.x * a.w) / 2 : w2;  // row stride in double2
    if (a.variant == 0) {
        double2* ring = reinterpret_cast<double2*>(smem);
        const int per = 2 * w2;  // wait: per half-entry only w2 items (W and T chunk per item)
        for (int ps = 0; ps < a.passes; ++ps) {
            const int2* E = a.ent + (size_t)ps * a.nh;
            const double* D = a.dd + (size_t)ps * a.nh;
            const int items = a.nh * w2;
            const int nmine = items > tid ? (items - tid + kThreads - 1) / kThreads : 0;
            int ii = tid, ic = tid;
            int si = 0, sc = 0;
            auto issue = [&]() {
                const int e = ii / w2, j2 = ii - e * w2;
                const int2 rs = __ldg(E + e);
                double2* slot = ring + (size_t)(si * 2) * kThreads + tid;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(slot)),
                             "l"(reinterpret_cast<const double2*>(Wb) + (long long)rs.x * ld2 + j2)
                             : "memory");
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(slot + kThreads)),
                             "l"(reinterpret_cast<const double2*>(Tb) + (long long)rs.y * ld2 + j2)
                             : "memory");
                asm volatile("cp.async.commit_group;" ::: "memory");
                si = (si + 1 == a.S) ? 0 : si + 1;
                ii += kThreads;
            };
            int ni = min(nmine, a.S - 1);
            for (int i = 0; i < ni; ++i) issue();
            for (int j = 0; j < nmine; ++j) {
                if (ni < nmine) {
                    issue();
                    ++ni;
                    if (a.S == 6) asm volatile("cp.async.wait_group 5;" ::: "memory");
                    else if (a.S == 8) asm volatile("cp.async.wait_group 7;" ::: "memory");
                    else asm volatile("cp.async.wait_group 11;" ::: "memory");
                } else {
                    asm volatile("cp.async.wait_group 0;" ::: "memory");
                }
                const int e = ic / w2, j2 = ic - e * w2;
                const int2 rs = __ldg(E + e);
                const double2* slot = ring + (size_t)(sc * 2) * kThreads + tid;
                double2 wv = slot[0];
                const double2 tv = slot[kThreads];
                const double d = __ldg(D + e);
                wv.x = fma(d, tv.x, wv.x);
                wv.y = fma(d, tv.y, wv.y);
                reinterpret_cast<double2*>(Wb)[(long long)rs.x * ld2 + j2] = wv;
                sc = (sc + 1 == a.S) ? 0 : sc + 1;
                ic += kThreads;
            }
            (void)per;
            __syncthreads();
        }
        return;
    }
    // per-warp bulk ring: Rw slots of (W row, T row), one mbarrier per slot
    const int Rw = a.Rw;
    const unsigned rowb = (unsigned)w * 8u;
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem) + (size_t)warp * Rw;
    const size_t soff = ((size_t)kWarps * Rw * 8 + 127) & ~(size_t)127;
    double* slots = reinterpret_cast<double*>(smem + soff) + (size_t)warp * Rw * 2 * w;
    if (lane == 0)
        for (int s = 0; s < Rw; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    unsigned phase_bits = 0;  // parity per slot (Rw <= 32)
    for (int ps = 0; ps < a.passes; ++ps) {
        const int2* E = a.ent + (size_t)ps * a.nh;
        const double* D = a.dd + (size_t)ps * a.nh;
        const int nmine = a.nh > warp ? (a.nh - warp + kWarps - 1) / kWarps : 0;
        auto issue = [&](int k) {  // k-th half-entry of this warp -> slot k % Rw
            const int s = k % Rw;
            const int e = warp + k * kWarps;
            const int2 rs = __ldg(E + e);
            double* sw = slots + (size_t)s * 2 * w;
            if (lane == 0) {
                if (a.variant == 3) {
                    mbar_expect_tx(bars + s, rowb);
                    bulk_g2s(sw + w, Tb + (long long)rs.y * w, rowb, bars + s);
                } else {
                    mbar_expect_tx(bars + s, 2 * rowb);
                    bulk_g2s(sw, Wb + (long long)rs.x * w, rowb, bars + s);
                    bulk_g2s(sw + w, Tb + (long long)rs.y * w, rowb, bars + s);
                }
            }
        };
        const int pre = min(nmine, Rw);
        for (int k = 0; k < pre; ++k) issue(k);
        double2 wnext = make_double2(0.0, 0.0);
        if (a.variant == 3 && nmine > 0 && lane < w2) {
            const int2 rs = __ldg(E + warp);
            wnext = __ldcg(reinterpret_cast<const double2*>(Wb + (long long)rs.x * w) + lane);
        }
        for (int k = 0; k < nmine; ++k) {
            const int s = k % Rw;
            const int e = warp + k * kWarps;
            const int2 rs = __ldg(E + e);
            const double d = __ldg(D + e);
            double2 wcur = wnext;
            if (a.variant == 3 && k + 1 < nmine && lane < w2) {
                const int2 rn = __ldg(E + e + kWarps);
                wnext = __ldcg(reinterpret_cast<const double2*>(Wb + (long long)rn.x * w) + lane);
            }
            mbar_wait(bars + s, (phase_bits >> s) & 1u);
            phase_bits ^= 1u << s;
            const double2* sw = reinterpret_cast<const double2*>(slots + (size_t)s * 2 * w);
            for (int j = lane; j < w2; j += 32) {
                double2 wv = (a.variant == 3) ? wcur : sw[j];
                const double2 tv = sw[w2 + j];
                wv.x = fma(d, tv.x, wv.x);
                wv.y = fma(d, tv.y, wv.y);
                reinterpret_cast<double2*>(Wb + (long long)rs.x * w)[j] = wv;
            }
            if (a.variant == 2) asm volatile("fence.proxy.async.global;" ::: "memory");
            __syncwarp();
            if (k + Rw < nmine) issue(k + Rw);
        }
        if (a.variant == 1 || a.variant == 3) asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncthreads();
    }
}

int main(int argc, char** argv) {
    int nsm_dev;
    cudaDeviceGetAttribute(&nsm_dev, cudaDevAttrMultiProcessorCount, 0);
    const int p = 5000;
    const int passes = 200;
    struct Cfg {
        int nsm, w, nh, rowmajor;
    } cfgs[] = {{148, 34, 484, 0},  {148, 34, 1936, 0}, {148, 34, 4840, 0}, {148, 36, 484, 0}, {148, 36, 1936, 0},
                {148, 34, 484, 1},  {148, 34, 1936, 1}, {148, 36, 484, 1},  {148, 36, 1936, 1}, {66, 76, 484, 0},
                {66, 76, 1936, 0},  {66, 76, 484, 1},   {66, 76, 1936, 1},  {41, 122, 484, 0}, {41, 122, 1936, 1}};
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
        srand(1);
        int* perm = (int*)malloc(sizeof(int) * p);
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
        struct V {
            int variant, S, Rw;
        } vs[] = {{0, 6, 0}, {0, 8, 0}, {0, 12, 0}, {1, 0, 8}};
        for (auto v : vs) {
            if (cf.rowmajor && v.variant != 0) continue;
            Args a{W, T, ent, dd, p, w, nh, passes, v.S, v.Rw, v.variant, slab, cf.rowmajor};
            size_t sm = v.variant == 0 ? (size_t)v.S * 2 * kThreads * 16
                                       : (((size_t)kWarps * v.Rw * 8 + 127) & ~(size_t)127) + (size_t)kWarps * v.Rw * 16 * w;
            if (v.variant == 3 && w / 2 > 32) continue;
            if (sm > 227 * 1024) {
                printf("nsm=%d w=%d variant=%d Rw=%d: smem %zu too large\n", nsm, w, v.variant, v.Rw, sm);
                continue;
            }
            cudaFuncSetAttribute(rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            rows_kernel<<<nsm, kThreads, sm>>>(a);
            cudaEventRecord(e0);
            rows_kernel<<<nsm, kThreads, sm>>>(a);
            cudaEventRecord(e1);
            cudaError_t err = cudaEventSynchronize(e1);
            if (err != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(err));
                return 1;
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double bytes = 24.0 * w * (double)nh * passes * nsm;
            printf("nsm=%3d w=%3d nh=%4d %s variant=%d S=%2d Rw=%2d smem=%6zu  %.3f ms  %.1f GB/s device  %.1f GB/s/SM  %.2f us/pass\n",
                   nsm, w, nh, cf.rowmajor ? "rowmajor" : "slab    ", v.variant, v.S, v.Rw, sm, ms, bytes / ms / 1e6, bytes / ms / 1e6 / nsm, 1e3 * ms / passes);
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
