// Dev microbenchmark: tcgen05.mma issue cost from one divergent thread (lane 0
// under `if`) vs a whole warp issuing through elect.sync (warp-uniform control
// flow, descriptors in uniform registers).  M=128, K=16 bf16, operands resident
// in smem, back-to-back chain into one accumulator; plus the per-k-block shape
// of the persistent kernel (4 MMAs + commit per stage, descriptor arithmetic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_issue tools/mma_issue.cu
#include <cstdio>
#include "../paper_2605_08975_b200/csrc/common.cuh"
using namespace alpa;

__device__ inline void tc_mma_bf16_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p, e;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ inline void tc_commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n"
        ".reg .pred e;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
        "}\n" ::"r"(smem_u32(bar))
        : "memory");
}

template <int N, int MODE>
__global__ void __launch_bounds__(128, 1) k(int iters, long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    uint8_t* A = smem;          // 4 stages of 128 rows x 64 k (SW128 K-major)
    uint8_t* B = smem + 65536;  // 4 stages of N rows x 64 k
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536 + 4 * 256 * 128);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 8);
    for (int i = threadIdx.x; i < (65536 + 4 * N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 5; ++s) mbar_init(bar + s, 1);
        fence_mbar_init();
    }
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(slot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = *slot;
    const uint32_t idesc = idesc_bf16(128, N);
    fence_proxy_async();
    if (MODE == 0 && threadIdx.x == 32) {
        // single divergent thread, stage-rotating descriptors (the kernel's pattern)
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int st = i & 3;
            const uint64_t da = sdesc_k_sw128(A + st * 16384), db = sdesc_k_sw128(B + st * N * 128);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) tc_mma_bf16(tb, da + 2 * kk, db + 2 * kk, idesc, (i | kk) ? 1u : 0u);
            tc_commit(bar + st);
        }
        tc_commit(bar + 4);
        mbar_wait(bar + 4, 0);
        const long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    } else if (MODE == 1 && warp == 1) {
        // whole warp, elect.sync inside the issuing asm
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int st = i & 3;
            const uint64_t da = sdesc_k_sw128(A + st * 16384), db = sdesc_k_sw128(B + st * N * 128);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) tc_mma_bf16_elect(tb, da + 2 * kk, db + 2 * kk, idesc, (i | kk) ? 1u : 0u);
            tc_commit_elect(bar + st);
        }
        tc_commit_elect(bar + 4);
        mbar_wait(bar + 4, 0);
        const long long t1 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 32) out[0] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 256);
}

template <int N, int MODE>
void run(long long* d) {
    const int smem = 65536 + 4 * 256 * 128 + 1024 + 128;
    cudaFuncSetAttribute(k<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    k<N, MODE><<<148, 128, smem>>>(iters, d);
    k<N, MODE><<<148, 128, smem>>>(iters, d);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double per = (double)c / (iters * 4.0);
    printf("%s N=%3d: %6.1f cycles/MMA  %5.0f%% of 8192 flop/clk  %s\n", MODE ? "warp+elect " : "one thread ", N, per,
           100.0 * 2.0 * 128 * N * 16 / per / 8192.0, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    run<16, 0>(d);
    run<16, 1>(d);
    run<32, 0>(d);
    run<32, 1>(d);
    run<64, 0>(d);
    run<64, 1>(d);
    run<128, 0>(d);
    run<128, 1>(d);
    run<192, 0>(d);
    run<192, 1>(d);
    run<256, 0>(d);
    run<256, 1>(d);
    return 0;
}
