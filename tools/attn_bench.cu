// Dev microbenchmark: the persistent kernel's attention block pipeline in
// isolation -- one MMA-issuer warp (whole warp, elected issue: S = Q K^T into two
// TMEM S buffers, PV into two key-half O accumulators) and the 8 softmax warps
// with the kernel's exact per-block protocol (s_full / s_free / p_full / p_free
// mbarriers), K/V and Q resident in smem (no TMA).  Cycles per 64-key block, to
// compare with the in-situ ~1650 (tools/attn_clk.py) and the softmax alone
// (tools/softmax_bench.cu).  Variants drop pieces of the pipeline.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/attn_bench tools/attn_bench.cu
#include <cstdio>
#include "../paper_2605_08975_b200/csrc/common.cuh"
using namespace alpa;

constexpr int HD = 128;
constexpr int KPANEL = 64 * 64 * 2, QPANEL = 128 * 64 * 2, KVB = 64 * HD * 2, P_BYTES = 128 * 64 * 2;
constexpr int STAGES = 4;
constexpr int OFF_Q = 0, OFF_KV = OFF_Q + 128 * HD * 2, OFF_P = OFF_KV + STAGES * 2 * KVB, OFF_BAR = OFF_P + 2 * P_BYTES;
constexpr int SMEM = OFF_BAR + 1024 + 1024;

// D (+)= A[tmem] . B[smem]: the A operand (128 rows x 16 bf16 = 8 packed columns) from TMEM
__device__ inline void tc_mma_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p, e;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ inline bool mbar_test_b(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(phase) : "memory");
    return ok != 0;
}
template <int MODE>
__device__ inline void wait_sm(uint64_t* bar, uint32_t phase) {
    if (MODE == 7) { while (!mbar_test_b(bar, phase)) {} }
    else mbar_wait(bar, phase);
}
__device__ inline void tc_mma_w(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) { tc_mma_bf16_w(d, a, b, id, acc); }

template <int MODE>  // 0: full pipeline; 1: no PV MMA (P published, no O); 2: softmax skips exps; 6: P in TMEM (TS MMA);
                     // 3: four S buffers, S issued three blocks ahead of PV
__global__ void __launch_bounds__(384, 1) k(int nblk, long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* s_full = bars;
    uint64_t* s_free = bars + 2;
    uint64_t* p_full = bars + 4;
    uint64_t* p_free = bars + 6;
    uint64_t* done = bars + 8;
    uint64_t* s_full4 = bars + 9;   // [4] (MODE 3)
    uint64_t* s_free4 = bars + 13;  // [4]
    uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 24);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // small pseudo-random bf16 operands (scores of O(1))
    for (int i = threadIdx.x; i < OFF_BAR / 2; i += blockDim.x) {
        const uint32_t h = (uint32_t)i * 2654435761u;
        reinterpret_cast<__nv_bfloat16*>(smem)[i] = __float2bfloat16(((int)(h >> 24) - 128) * (1.0f / 512.0f));
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_free[i], 8);
            mbar_init(&p_full[i], 8);
            mbar_init(&p_free[i], 1);
        }
        mbar_init(done, 1);
        for (int i = 0; i < 4; ++i) {
            mbar_init(&s_full4[i], 1);
            mbar_init(&s_free4[i], 8);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(slot, 512);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *slot;
    const uint32_t tS[2] = {tbase, tbase + 64};
    const uint32_t tO[2] = {tbase + 128, tbase + 128 + HD};
    const uint32_t tS4[4] = {tbase, tbase + 64, tbase + 384, tbase + 448};  // MODE 3 (O at 128..383)
    const uint32_t tP[2] = {tbase + 384, tbase + 416};                     // MODE 6: P (32 packed cols)
    if (warp == 1) {
        constexpr uint32_t idS = idesc_bf16(128, 64);
        constexpr uint32_t idO = idesc_bf16(128, HD, true);
        auto issue_pv = [&](int j) {
            mbar_wait(&p_full[j & 1], (j >> 1) & 1);
            tc_fence_after();
            if (MODE == 6) {
                const uint8_t* vb = smem + OFF_KV + (j % STAGES) * 2 * KVB + KVB;
#pragma unroll
                for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) {
                        const int ks16 = hh * 2 + kk;
                        tc_mma_ts_w(tO[hh], tP[j & 1] + ks16 * 8, sdesc_mn_sw128(vb + ks16 * 2048, KPANEL), idO,
                                    (j == 0 && kk == 0) ? 0u : 1u);
                    }
            } else if (MODE != 1) {
                const uint8_t* pb = smem + OFF_P + (j & 1) * P_BYTES;
                const uint8_t* vb = smem + OFF_KV + (j % STAGES) * 2 * KVB + KVB;
#pragma unroll
                for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) {
                        const int ks16 = hh * 2 + kk;
                        tc_mma_w(tO[hh], sdesc_k_sw128(pb) + 2 * ks16, sdesc_mn_sw128(vb + ks16 * 2048, KPANEL), idO,
                                 (j == 0 && kk == 0) ? 0u : 1u);
                    }
            }
            tc_commit_w(&p_free[j & 1]);
        };
        auto issue_s4 = [&](int j) {
            if (j >= 4) mbar_wait(&s_free4[j & 3], ((j - 4) >> 2) & 1);
            tc_fence_after();
            const uint8_t* kb = smem + OFF_KV + (j % STAGES) * 2 * KVB;
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk)
                tc_mma_w(tS4[j & 3], sdesc_k_sw128(smem + OFF_Q + (kk >> 2) * QPANEL) + 2 * (kk & 3),
                         sdesc_k_sw128(kb + (kk >> 2) * KPANEL) + 2 * (kk & 3), idS, kk > 0 ? 1u : 0u);
            tc_commit_w(&s_full4[j & 3]);
        };
        if (MODE == 3 || MODE == 4) {
            issue_s4(0);
            issue_s4(1);
            issue_s4(2);
            for (int j = 0; j < nblk; ++j) {
                if (MODE == 3 && j + 3 < nblk) issue_s4(j + 3);
                issue_pv(j);
                if (MODE == 4 && j + 3 < nblk) issue_s4(j + 3);
            }
        } else if (MODE == 5) {  // 4 S buffers, S two blocks ahead (ring lookahead 1)
            issue_s4(0);
            issue_s4(1);
            for (int j = 0; j < nblk; ++j) {
                if (j + 2 < nblk) issue_s4(j + 2);
                issue_pv(j);
            }
        } else {
        for (int j = 0; j < nblk; ++j) {
            if (j >= 2) mbar_wait(&s_free[j & 1], ((j - 2) >> 1) & 1);
            tc_fence_after();
            const uint8_t* kb = smem + OFF_KV + (j % STAGES) * 2 * KVB;
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk)
                tc_mma_w(tS[j & 1], sdesc_k_sw128(smem + OFF_Q + (kk >> 2) * QPANEL) + 2 * (kk & 3),
                         sdesc_k_sw128(kb + (kk >> 2) * KPANEL) + 2 * (kk & 3), idS, kk > 0 ? 1u : 0u);
            tc_commit_w(&s_full[j & 1]);
            if (j > 0) issue_pv(j - 1);
        }
        issue_pv(nblk - 1);
        }
        tc_commit_w(done);
    } else if (warp >= 4) {
        const int q = warp & 3, hh = (warp - 4) >> 2, i = q * 32 + lane;
        const uint32_t lane_off = uint32_t(q * 32) << 16;
        const uint32_t tOh = tbase + 128 + hh * HD;
        const float sl2 = 0.0883883f * 1.4426950408889634f;
        float m_ref = -INFINITY, l = 0.f;
        long long t0 = 0;
        for (int j = 0; j < nblk; ++j) {
            if (j == 8) t0 = clock64();
            const int b = j & 1;
            const bool st = blockIdx.x == 0 && threadIdx.x == 128 && j >= 100 && j < 104;
            long long* so = out + 2 + (j - 100) * 8;
            if (st) so[0] = clock64();
            if (MODE >= 3 && MODE <= 5) mbar_wait(&s_full4[j & 3], (j >> 2) & 1);
            else wait_sm<MODE>(&s_full[b], (j >> 1) & 1);
            if (st) so[1] = clock64();
            tc_fence_after();
            uint32_t sr[32];
            tmem_ld32((MODE >= 3 && MODE <= 5 ? tS4[j & 3] : tS[b]) + lane_off + hh * 32, sr);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(MODE >= 3 && MODE <= 5 ? &s_free4[j & 3] : &s_free[b]);
            const float* srf = reinterpret_cast<const float*>(sr);
            float t8[8];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                t8[kk] = fmaxf(fmaxf(srf[4 * kk], srf[4 * kk + 1]), fmaxf(srf[4 * kk + 2], srf[4 * kk + 3]));
            const float mx = fmaxf(fmaxf(fmaxf(t8[0], t8[1]), fmaxf(t8[2], t8[3])),
                                   fmaxf(fmaxf(t8[4], t8[5]), fmaxf(t8[6], t8[7]))) * sl2;
            float corr = 1.f;
            if (m_ref == -INFINITY) m_ref = mx;
            else if (mx > m_ref + 8.f) { corr = ex2(m_ref - mx); m_ref = mx; }
            const float nb = -m_ref;
            float r4[4] = {0.f, 0.f, 0.f, 0.f};
            uint32_t pk[16];
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
                float p0, p1;
                if (MODE == 2) {
                    p0 = fmaf(srf[2 * kk], sl2, nb);
                    p1 = fmaf(srf[2 * kk + 1], sl2, nb);
                } else {
                    p0 = ex2(fmaf(srf[2 * kk], sl2, nb));
                    p1 = ex2(fmaf(srf[2 * kk + 1], sl2, nb));
                }
                r4[kk & 3] += p0 + p1;
                pk[kk] = pack_bf16x2(p0, p1);
            }
            l = l * corr + (r4[0] + r4[1]) + (r4[2] + r4[3]);
            if (st) so[2] = clock64();
            if (j >= 2) wait_sm<MODE>(&p_free[b], ((j - 2) >> 1) & 1);
            if (st) so[3] = clock64();
            if (MODE == 6) {
                tmem_st16(tP[b] + lane_off + hh * 16, pk);
                tmem_st_wait();
            } else {
            uint8_t* prow = smem + OFF_P + b * P_BYTES + i * 128;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int ch = hh * 4 + c;
                *reinterpret_cast<uint4*>(prow + ((ch ^ (i & 7)) << 4)) =
                    make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
            }
            fence_proxy_async();
            }
            if (__any_sync(0xffffffffu, corr != 1.f)) {
                if (j >= 1) mbar_wait(&p_free[(j - 1) & 1], ((j - 1) >> 1) & 1);
                tc_fence_after();
#pragma unroll 1
                for (int cc = 0; cc < HD; cc += 32) {
                    uint32_t ov[32];
                    tmem_ld32(tOh + lane_off + cc, ov);
                    tmem_ld_wait();
#pragma unroll
                    for (int e2 = 0; e2 < 32; ++e2) ov[e2] = __float_as_uint(__uint_as_float(ov[e2]) * corr);
                    tmem_st32(tOh + lane_off + cc, ov);
                }
                tmem_st_wait();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[b]);
            if (st) so[4] = clock64();
        }
        const long long t1 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 128) out[0] = (t1 - t0);
        if (l == 12345.f) out[1] = 1;
    }
    if (warp == 1) mbar_wait(done, 0);
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tbase, 512);
}

template <int MODE>
void run(long long* d, const char* name) {
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    const int nblk = 2008;
    k<MODE><<<148, 384, SMEM>>>(nblk, d);
    k<MODE><<<148, 384, SMEM>>>(nblk, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("%-34s %7.1f cycles per 64-key block  %s\n", name, (double)c / (nblk - 8), cudaGetErrorString(e));
    fflush(stdout);
}

int main(int argc, char** argv) {
    long long* d;
    cudaMalloc(&d, 64 * 8);
    if (argc > 1 && (atoi(argv[1]) == 9 || atoi(argv[1]) == 7)) {  // stamped run of the default pipeline
        if (atoi(argv[1]) == 9) run<0>(d, "full pipeline (stamped)");
        else run<7>(d, "softmax waits by test_wait polling");
        long long h[64];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        for (int b = 0; b < 4; ++b) {
            long long* so = h + 2 + b * 8;
            printf("block %d: wait S %lld  S->exps done %lld  P slot wait %lld  P store+fence+arrive %lld  (total %lld)\n", b,
                   so[1] - so[0], so[2] - so[1], so[3] - so[2], so[4] - so[3], so[4] - so[0]);
        }
        return 0;
    }
    if (argc > 1) {  // one variant
        const int m = atoi(argv[1]);
        if (m == 6) run<6>(d, "P in TMEM (TS MMA for PV)");
        return 0;
    }
    run<0>(d, "full pipeline (S, softmax, PV)");
    run<1>(d, "no PV MMA");
    run<2>(d, "softmax without exps");
    run<3>(d, "4 S buffers, S 3 blocks ahead");
    run<4>(d, "4 S buffers, PV_j then S_{j+3}");
    run<5>(d, "4 S buffers, S 2 blocks ahead");
    return 0;
}
