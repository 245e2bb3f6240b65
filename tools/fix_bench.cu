// Dev microbenchmark: mk::fix_t (split-K finalisation in the TMEM layout) in
// isolation: 128 CTAs, S=4, 24 owned tokens per warp half, MLP2 shapes.
#include <cstdio>
#include "../paper_2605_08975_b200/csrc/mk.cuh"
using namespace alpa;
using namespace alpa::mk;

__global__ void __launch_bounds__(320, 1) fix_kernel(const float* ws, float* e, __nv_bfloat16* xb, int mode,
                                                     long long* out_cycles, int ld) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 1) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = slot;
    float2* st_part = reinterpret_cast<float2*>(smem);
    const int M = 384, nf = ld;
    const int tile = blockIdx.x / 4, s = blockIdx.x % 4;
    const int f0 = (tile % 16) * 128, t0 = (tile / 16) * 192;
    if (warp >= 2) {
        const int ew = warp - 2, q = warp & 3, hh = ew >> 2;
        const int own_lo = s * 48, my_lo = own_lo + hh * 24;
        const int f = f0 + q * 32 + lane;
        FixArgs fa;
        fa.tacc = tbase + ((uint32_t)(q * 32) << 16) + my_lo;
        fa.testage = tbase + ((uint32_t)(q * 32) << 16) + 256 + my_lo;
        fa.ncol = 24;
        fa.c0 = my_lo;
        fa.S = (mode & 1) ? 1 : 4;
        fa.s_own = (mode & 1) ? 0 : s;
        fa.ws = ws + (long long)(t0 + my_lo) * nf + f;
        fa.split_stride = (long long)M * nf;
        fa.nf = nf;
        fa.bf = 0.1f;
        fa.erow = e + (long long)(t0 + my_lo) * nf + f;
        fa.xrow = (mode & 2) ? nullptr : xb + (long long)(t0 + my_lo) * nf + f;
        fa.ldo = nf;
        fa.st_part = (mode & 4) ? nullptr : st_part;
        fa.q = q;
        fa.lane = lane;
        for (int rep = 0; rep < 4; ++rep) {
            asm volatile("bar.sync 1, 256;");
            const long long c0 = clock64();
            fix_t<true>(fa);
            asm volatile("bar.sync 1, 256;");
            const long long c1 = clock64();
            if (threadIdx.x == 64) out_cycles[blockIdx.x * 4 + rep] = c1 - c0;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tbase, 512);
}

int main() {
    float *ws, *e;
    __nv_bfloat16* xb;
    long long* d;
    cudaMalloc(&ws, (size_t)4 * 384 * 2080 * 4);
    cudaMalloc(&e, (size_t)384 * 2080 * 4);
    cudaMalloc(&xb, (size_t)384 * 2080 * 2);
    cudaMalloc(&d, 128 * 4 * 8);
    cudaMemset(ws, 0, (size_t)4 * 384 * 2080 * 4);
    cudaFuncSetAttribute(fix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int mode : {0, 7, 8, 15}) {
        fix_kernel<<<128, 320, 64 * 1024>>>(ws, e, xb, mode, d, (mode & 8) ? 2048 + 32 : 2048);
        cudaDeviceSynchronize();
        long long h[512];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double avg[4] = {0, 0, 0, 0};
        for (int b = 0; b < 128; ++b)
            for (int r = 0; r < 4; ++r) avg[r] += h[b * 4 + r] / 128.0;
        printf("mode %d (%s%s%s%s) cycles: first %6.0f then %6.0f %6.0f %6.0f (%s)\n", mode, mode & 1 ? "S=1 " : "S=4 ",
               mode & 2 ? "noXB " : "", mode & 4 ? "noStats " : "", mode & 8 ? "ld=2080" : "ld=2048", avg[0], avg[1], avg[2], avg[3],
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
