// Experiment: a 2-CTA (cta_group::2) tcgen05 MMA and a 1-CTA MMA in the same
// kernel / cluster, TMEM allocated per CTA with cta_group::1.  M=256 (pair),
// N=64, K=64; A, B K-major SW128 in smem (filled by threads, not TMA).
#include <cstdio>
#include "../paper_2605_08975_b200/csrc/common.cuh"
using namespace alpa;

__device__ inline void mma_cg2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ inline void commit_cg2_mc(uint64_t* bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(bar)), "h"(mask) : "memory");
}
__device__ inline void tmem_alloc2(uint32_t* dst, uint32_t n) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(n) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ inline void tmem_dealloc2(uint32_t a, uint32_t n) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(a), "r"(n) : "memory");
}

// element (row, k) of a K-major SW128 tile with 64-wide K (128 B rows)
__device__ inline int sw_off(int row, int k) { return row * 128 + ((((k >> 3) ^ (row & 7))) << 4) + (k & 7) * 2; }

template <int MODE>  // 0: alloc cg1 + mma cg2 ; 1: alloc cg2 + mma cg2 ; 2: alloc cg1, mma cg2 then cg1
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(float* out, int* flag) {
    __shared__ __align__(1024) uint8_t A[128 * 128];  // this CTA's 128 rows of A (256 total), K=64
    __shared__ __align__(1024) uint8_t B[32 * 128];   // this CTA's 32 of N=64 columns of B
    __shared__ __align__(1024) uint8_t B1[64 * 128];  // full B for the 1-CTA MMA
    __shared__ uint64_t bar, bar1;
    __shared__ uint32_t slot;
    const uint32_t rank = cluster_ctarank();
    const int tid = threadIdx.x;
    // A[m][k] = (m_global % 7 - 3) * 0.25, B[n][k] = ((n + k) % 5 - 2) * 0.5 (n global)
    for (int i = tid; i < 128 * 64; i += 128) {
        const int r = i / 64, kk = i % 64, mg = rank * 128 + r;
        *reinterpret_cast<__nv_bfloat16*>(A + sw_off(r, kk)) = __float2bfloat16((mg % 7 - 3) * 0.25f);
    }
    for (int i = tid; i < 32 * 64; i += 128) {
        const int r = i / 64, kk = i % 64, ng = rank * 32 + r;
        *reinterpret_cast<__nv_bfloat16*>(B + sw_off(r, kk)) = __float2bfloat16(((ng + kk) % 5 - 2) * 0.5f);
    }
    for (int i = tid; i < 64 * 64; i += 128) {
        const int r = i / 64, kk = i % 64;
        *reinterpret_cast<__nv_bfloat16*>(B1 + sw_off(r, kk)) = __float2bfloat16(((r + kk) % 5 - 2) * 0.5f);
    }
    if (tid == 0) { mbar_init(&bar, 1); mbar_init(&bar1, 1); fence_mbar_init(); }
    fence_proxy_async();
    if (tid < 32) { if (MODE == 1) tmem_alloc2(&slot, 128); else tmem_alloc(&slot, 128); }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tb = slot;
    if (rank == 0 && tid == 0) {
        const uint32_t idesc = idesc_bf16(256, 64);
        for (int kk = 0; kk < 4; ++kk)
            mma_cg2(tb, sdesc_k_sw128(A) + 2 * kk, sdesc_k_sw128(B) + 2 * kk, idesc, kk > 0);
        commit_cg2_mc(&bar, 3);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    // each CTA: TMEM lanes = its 128 rows, columns 0..63 = N
    const int warp = tid >> 5, lane = tid & 31;
    uint32_t r[16];
    for (int c = 0; c < 64; c += 16) {
        tmem_ld16(tb + ((uint32_t)(warp * 32) << 16) + c, r);
        tmem_ld_wait();
        for (int j = 0; j < 16; ++j) out[((rank * 128 + warp * 32 + lane) * 64) + c + j] = __uint_as_float(r[j]);
    }
    if (MODE == 2) {
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        if (tid == 0) {
            const uint32_t idesc = idesc_bf16(128, 64);
            for (int kk = 0; kk < 4; ++kk)
                tc_mma_bf16(tb + 64, sdesc_k_sw128(A) + 2 * kk, sdesc_k_sw128(B1) + 2 * kk, idesc, kk > 0);
            tc_commit(&bar1);
        }
        mbar_wait(&bar1, 0);
        tc_fence_after();
        for (int c = 0; c < 64; c += 16) {
            tmem_ld16(tb + ((uint32_t)(warp * 32) << 16) + 64 + c, r);
            tmem_ld_wait();
            for (int j = 0; j < 16; ++j) out[256 * 64 + ((rank * 128 + warp * 32 + lane) * 64) + c + j] = __uint_as_float(r[j]);
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (tid < 32) { if (MODE == 1) tmem_dealloc2(tb, 128); else tmem_dealloc(tb, 128); }
}

int main() {
    float* d;
    int* f;
    cudaMalloc(&d, 2 * 256 * 64 * 4);
    cudaMalloc(&f, 4);
    float h[2 * 256 * 64];
    for (int mode = 0; mode < 3; ++mode) {
        cudaMemset(d, 0, sizeof(h));
        if (mode == 0) k<0><<<2, 128>>>(d, f);
        if (mode == 1) k<1><<<2, 128>>>(d, f);
        if (mode == 2) k<2><<<2, 128>>>(d, f);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double maxerr = 0, maxerr1 = 0;
        for (int m = 0; m < 256; ++m)
            for (int n = 0; n < 64; ++n) {
                double ref = 0, ref1 = 0;
                for (int kk = 0; kk < 64; ++kk) {
                    ref += ((m % 7 - 3) * 0.25) * (((n + kk) % 5 - 2) * 0.5);
                }
                maxerr = fmax(maxerr, fabs(h[m * 64 + n] - ref));
                ref1 = ref;  // 1-CTA MMA: rows of this CTA x full B -> same values
                if (mode == 2) maxerr1 = fmax(maxerr1, fabs(h[256 * 64 + m * 64 + n] - ref1));
            }
        printf("mode %d: %s  cg2 max err %.3g  cg1-after max err %.3g\n", mode, cudaGetErrorString(e), maxerr, maxerr1);
        if (e != cudaSuccess) break;
    }
    return 0;
}
