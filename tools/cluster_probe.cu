// Dev probe: how many clusters of size C of a 1-CTA-per-SM kernel (full smem)
// are co-resident, and whether a cooperative launch accepts a cluster dimension.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(384, 1) k(int* out) {
    extern __shared__ unsigned char sm[];
    sm[threadIdx.x] = 1;
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    if (threadIdx.x == 0) out[blockIdx.x] = (int)r;
}

int main() {
    const int smem = 227 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int* d;
    cudaMalloc(&d, 4096);
    for (int cs : {1, 2, 3, 4, 6, 8, 16}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cs * 16);
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
        printf("cluster %2d: max active clusters %d (%d CTAs) %s\n", cs, ncl, ncl * cs, cudaGetErrorString(e));
        // cooperative + cluster launch of exactly the co-resident grid
        if (ncl > 0) {
            at[1].id = cudaLaunchAttributeCooperative;
            at[1].val.cooperative = 1;
            cfg.numAttrs = 2;
            cfg.gridDim = dim3(ncl * cs);
            e = cudaLaunchKernelEx(&cfg, k, d);
            cudaError_t e2 = cudaDeviceSynchronize();
            printf("   cooperative launch grid %d: %s / %s\n", ncl * cs, cudaGetErrorString(e), cudaGetErrorString(e2));
            cudaGetLastError();
        }
    }
    return 0;
}
