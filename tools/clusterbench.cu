// Floor of a cluster-resident colour chain: per phase, every CTA of one
// cluster pushes its P/CS published values (16 B each) into the owning CTA's
// shared memory through DSMEM, barrier.cluster, reads them back, barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/clusterbench tools/clusterbench.cu
// Also reports how many CTAs a cooperative launch with clusters can keep resident.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdio.h>

namespace cg = cooperative_groups;

__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(512, 1)
    phase_kernel(int P, int phases, int two_bar, double* sink) {
    extern __shared__ double2 inbox[];  // [P / 8] values this CTA owns
    cg::cluster_group cl = cg::this_cluster();
    const int cs = cl.num_blocks(), me = cl.block_rank();
    const int per = (P + cs - 1) / cs;
    double acc = 0.0;
    for (int g = 0; g < phases; ++g) {
        // publish: column c (own) pushes to the owner of its partner (a permutation changing per phase)
        for (int j = threadIdx.x; j < per; j += blockDim.x) {
            const int c = me * per + j;
            if (c >= P) break;
            const int dst = (int)(((unsigned)c * 2654435761u + (unsigned)g * 40503u) % (unsigned)P);
            const int owner = dst / per, slot = dst - owner * per;
            double2* remote = cl.map_shared_rank(inbox, owner);
            remote[slot] = make_double2(acc + c, (double)g);
        }
        if (two_bar) cl.sync();
        // consume: read own inbox (as the closed forms would)
        for (int j = threadIdx.x; j < per; j += blockDim.x) acc += inbox[j].x * 1e-30;
        cl.sync();
    }
    if (acc == 1.2345) sink[0] = acc;
}

__global__ void dummy_kernel(int* x) {
    if (x) x[0] = 0;
}

int main() {
    double* sink;
    cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int P : {5000, 20000}) {
        for (int two : {1, 0}) {
            const int per = (P + 7) / 8;
            const size_t smem = sizeof(double2) * per;
            cudaFuncSetAttribute(phase_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            const int phases = 20000;
            cudaEventRecord(e0);
            phase_kernel<<<8, 512, smem>>>(P, phases, two, sink);
            cudaEventRecord(e1);
            cudaError_t e = cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("P=%5d barriers/phase=%d : %s %.3f us/phase\n", P, two ? 2 : 1, cudaGetErrorString(e),
                   ms * 1e3 / phases);
        }
    }
    // co-residency of a cooperative launch with clusters of 8, 512 threads, 100 KB smem
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 8;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = 100 * 1024;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaFuncSetAttribute(dummy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int cs : {2, 4, 8, 16}) {
        attr[0].val.clusterDim.x = cs;
        if (cs == 16) cudaFuncSetAttribute(dummy_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cfg.gridDim = dim3(cs * 16);
        int nclusters = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, dummy_kernel, &cfg);
        printf("cluster=%2d: max active clusters %d (%d CTAs) %s\n", cs, nclusters, nclusters * cs,
               cudaGetErrorString(e));
        cfg.numAttrs = 2;
        cfg.gridDim = dim3(nclusters * cs);
        e = cudaLaunchKernelEx(&cfg, dummy_kernel, (int*)nullptr);
        cudaError_t e2 = cudaDeviceSynchronize();
        printf("          cooperative launch of %d CTAs: %s / %s\n", nclusters * cs, cudaGetErrorString(e),
               cudaGetErrorString(e2));
        cfg.numAttrs = 1;
    }
    return 0;
}
