// Dev microbenchmark: the persistent kernel's generic drain (mk::drain) in
// isolation: 128 CTAs, TMEM allocated, MLP1-shaped tile (TN 192, 8 epilogue
// warps), timed per call with clock64 (first = cold, then warm repeats).
#include <cstdio>
#include "../paper_2605_08975_b200/csrc/mk.cuh"
using namespace alpa;
using namespace alpa::mk;

__global__ void __launch_bounds__(320, 1) drain_kernel(int mode, long long* out_cycles, float* gout) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 1) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = slot;
    float* mu_s = reinterpret_cast<float*>(smem + 64 * 1024);
    float* rs_s = mu_s + 256;
    float2* st_part = reinterpret_cast<float2*>(rs_s + 256);
    if (threadIdx.x < 256) { mu_s[threadIdx.x] = 0.01f; rs_s[threadIdx.x] = 1.1f; }
    __syncthreads();
    if (warp >= 2) {
        const int ew = warp - 2, q = warp & 3, hh = ew >> 2;
        const int cb = hh * 96;
        DrainArgs da;
        da.tacc = tbase + ((uint32_t)(q * 32) << 16) + cb;
        da.tres = tbase + ((uint32_t)(q * 32) << 16) + 256 + cb;
        da.ncol = 96;
        da.nvalid = 96;
        da.cb = cb;
        da.q = q;
        da.lane = lane;
        for (int k = 0; k < 4; ++k) { da.bf[k] = 0.1f * k; da.cs[k] = 0.5f; }
        da.mu_s = mu_s;
        da.rs_s = rs_s;
        da.eout = (mode & 8) ? gout + (size_t)blockIdx.x * 192 * 2048 + q * 32 : nullptr;
        da.ldo = 2048;
        da.stg = smem;
        da.tn = 192;
        da.st_part = st_part;
        for (int rep = 0; rep < 4; ++rep) {
            asm volatile("bar.sync 1, 256;");
            const long long t0 = clock64();
            drain(da, mode & 2, mode & 1, mode & 4, mode & 8, mode & 8);
            asm volatile("bar.sync 1, 256;");
            const long long t1 = clock64();
            if (threadIdx.x == 64) out_cycles[blockIdx.x * 4 + rep] = t1 - t0;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tbase, 512);
}

int main() {
    long long* d;
    float* g;
    cudaMalloc(&d, 128 * 4 * 8);
    cudaMalloc(&g, (size_t)128 * 192 * 2048 * 4);
    cudaFuncSetAttribute(drain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    
    for (int mode : {0, 1, 2, 3, 12}) {
        drain_kernel<<<128, 320, 100 * 1024>>>(mode, d, g);
        cudaDeviceSynchronize();
        long long h[512];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double avg[4] = {0, 0, 0, 0};
        for (int b = 0; b < 128; ++b)
            for (int r = 0; r < 4; ++r) avg[r] += h[b * 4 + r] / 128.0;
        printf("mode %2d (%s%s%s%s) cycles: first %6.0f  then %6.0f %6.0f %6.0f  (%s)\n", mode, mode & 16 ? "noTMEM " : "", mode & 32 ? "noSTS " : "", mode & 1 ? "gelu " : "", mode & 2 ? "ln" : "", avg[0], avg[1],
               avg[2], avg[3], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
