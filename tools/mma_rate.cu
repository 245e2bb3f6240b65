// Dev microbenchmark: tcgen05.mma (kind::f16, bf16, cta_group::1, M=128, K=16)
// issue rate vs N with operands resident in smem (no TMA): cycles per MMA for a
// long back-to-back chain into one accumulator, one CTA per SM on every SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_rate tools/mma_rate.cu
#include <cstdio>
#include "../paper_2605_08975_b200/csrc/common.cuh"
using namespace alpa;

template <int N>
__global__ void __launch_bounds__(128, 1) k(int iters, long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    uint8_t* A = smem;             // 128 rows x 64 k (16 KB, SW128 K-major)
    uint8_t* B = smem + 16384;     // N rows x 64 k
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 256 * 128);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(slot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = *slot;
    if (threadIdx.x == 32) {
        fence_proxy_async();
        const uint64_t da = sdesc_k_sw128(A), db = sdesc_k_sw128(B);
        const uint32_t idesc = idesc_bf16(128, N);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) tc_mma_bf16(tb, da + 2 * kk, db + 2 * kk, idesc, (i | kk) ? 1u : 0u);
        tc_commit(bar);
        mbar_wait(bar, 0);
        const long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 256);
}

template <int N>
void run(long long* d) {
    const int smem = 16384 + 256 * 128 + 1024 + 64;
    cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    k<N><<<148, 128, smem>>>(iters, d);
    k<N><<<148, 128, smem>>>(iters, d);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double per = (double)c / (iters * 4.0);
    printf("M=128 N=%3d K=16: %6.1f cycles/MMA  %7.0f flop/cycle/SM (%.0f%% of 8192)  %s\n", N, per,
           2.0 * 128 * N * 16 / per, 100.0 * 2.0 * 128 * N * 16 / per / 8192.0,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    run<32>(d);
    run<64>(d);
    run<96>(d);
    run<128>(d);
    run<160>(d);
    run<192>(d);
    run<256>(d);
    return 0;
}
