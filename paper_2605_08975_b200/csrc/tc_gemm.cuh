// tcgen05 / TMEM / TMA GEMM for the bf16 path (sm_100a).
//
//   out[t][f] (op)= sum_k X[t][k] * W[f][k] + bias[f]
//
// "Swap-AB" orientation: the weight tile (128 output features) is the MMA M
// operand and the token tile (TN <= 256 action tokens of all trajectories) is
// the MMA N operand, so every weight byte is streamed from HBM once per token
// tile while the tiny activation (M = 64 N rows) is re-read from L2.  The
// accumulator lives in TMEM (128 lanes = features, TN columns = tokens); the
// epilogue warps own one feature each, so stores of one token column are
// coalesced across the warp and bias is a per-thread scalar.
//
// Roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA
// issuer (one elected lane), warps 2..5 = epilogue (TMEM lane quarters
// 2,3,0,1).  Multi-stage smem ring with full/empty mbarriers.
//
// Split-K is deterministic: every split writes its partial tile, the last
// arriving CTA (tile counter) sums the partials in split order and applies
// the fused epilogue (bias / GELU / residual), then re-arms the counter.
#pragma once

#include "common.cuh"

namespace alpa {

enum Epi : int {
    EPI_BF16 = 0,       // out bf16 = acc + b                      (QKV, model.cpp:574-576)
    EPI_GELU_BF16 = 1,  // out bf16 = gelu(acc + b)                (mlp1 + gelu, model.cpp:585-586)
    EPI_F32 = 2,        // out f32  = acc + b                      (encoder mlp2, model.cpp:562)
    EPI_RESID_F32 = 3,  // out f32  = out + (acc + b)              (o / mlp2 + residual, model.cpp:582-588)
};

struct GemmArgs {
    int nf, t, k;          // features (MMA M), tokens (MMA N), reduction
    const float* bias;     // [nf]
    void* out;             // [t][ldo]
    int64_t ldo;
    int splits, kbs;       // split-K count, 64-wide k-blocks per split
    float* ws;             // [splits][t][nf] partials (splits > 1)
    int* counters;         // per output tile
};

template <int TN>
struct GemmCfg {
    static constexpr int W_BYTES = 128 * 64 * 2;
    static constexpr int X_BYTES = TN * 64 * 2;
    static constexpr int STAGE = W_BYTES + X_BYTES;
    static constexpr int STAGES = (200 * 1024) / STAGE > 8 ? 8 : (200 * 1024) / STAGE;
    static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
    static constexpr uint32_t TCOLS = TN <= 32 ? 32 : TN <= 64 ? 64 : TN <= 128 ? 128 : 256;
};

template <int EPI>
__device__ inline void epi_store(const GemmArgs& a, int t, int f, float v) {
    if constexpr (EPI == EPI_BF16) {
        reinterpret_cast<__nv_bfloat16*>(a.out)[(int64_t)t * a.ldo + f] = __float2bfloat16_rn(v);
    } else if constexpr (EPI == EPI_GELU_BF16) {
        reinterpret_cast<__nv_bfloat16*>(a.out)[(int64_t)t * a.ldo + f] =
            __float2bfloat16_rn(gelu_erf(v));
    } else if constexpr (EPI == EPI_F32) {
        reinterpret_cast<float*>(a.out)[(int64_t)t * a.ldo + f] = v;
    } else {
        float* o = reinterpret_cast<float*>(a.out) + (int64_t)t * a.ldo + f;
        *o = *o + v;
    }
}

template <int TN, int EPI>
__global__ void __launch_bounds__(192, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const GemmArgs a) {
    using C = GemmCfg<TN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
    uint64_t* empty = full + C::STAGES;
    uint64_t* accf = empty + C::STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);
    __shared__ int s_last;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int f0 = blockIdx.x * 128, t0 = blockIdx.y * TN;
    const int KB = a.k / 64;
    const int kb0 = blockIdx.z * a.kbs;
    const int nkb = min(KB, kb0 + a.kbs) - kb0;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmW);
        tma_prefetch(&tmX);
        for (int i = 0; i < C::STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(accf, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, C::TCOLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // Weights are independent of the previous kernel: prefetch the
            // first stages before waiting on the producer of X (PDL overlap).
            const int pre = nkb < C::STAGES ? nkb : C::STAGES;
            for (int i = 0; i < pre; ++i) {
                mbar_expect_tx(&full[i], C::STAGE);
                tma_load_2d(smem + i * C::STAGE, &tmW, &full[i], (kb0 + i) * 64, f0);
            }
            pdl_wait();
            for (int i = 0; i < nkb; ++i) {
                const int st = i % C::STAGES;
                const uint32_t ph = (i / C::STAGES) & 1;
                uint8_t* sw = smem + st * C::STAGE;
                if (i >= pre) {
                    mbar_wait(&empty[st], ph ^ 1);
                    mbar_expect_tx(&full[st], C::STAGE);
                    tma_load_2d(sw, &tmW, &full[st], (kb0 + i) * 64, f0);
                }
                tma_load_2d(sw + C::W_BYTES, &tmX, &full[st], (kb0 + i) * 64, t0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16(128, TN);
            for (int i = 0; i < nkb; ++i) {
                const int st = i % C::STAGES;
                const uint32_t ph = (i / C::STAGES) & 1;
                mbar_wait(&full[st], ph);
                tc_fence_after();
                uint8_t* sw = smem + st * C::STAGE;
                const uint64_t da = sdesc_k_sw128(sw);
                const uint64_t db = sdesc_k_sw128(sw + C::W_BYTES);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    tc_mma_bf16(tbase, da + 2 * k, db + 2 * k, idesc, (i | k) != 0 ? 1u : 0u);
                tc_commit(&empty[st]);
            }
            tc_commit(accf);
        }
        __syncwarp();
    } else {
        // ---------------- epilogue: warps 2..5 ----------------
        const int q = warp & 3;
        const int f = f0 + q * 32 + lane;
        const float bias = a.bias[f];
        const uint32_t trow = tbase + (uint32_t(q * 32) << 16);
        mbar_wait(accf, 0);
        tc_fence_after();
        pdl_launch();
        if (a.splits == 1) {
            for (int c = 0; c < TN; c += 16) {
                uint32_t r[16];
                tmem_ld16(trow + c, r);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int t = t0 + c + j;
                    if (t < a.t) epi_store<EPI>(a, t, f, __uint_as_float(r[j]) + bias);
                }
            }
        } else {
            float* wsz = a.ws + (size_t)blockIdx.z * a.t * a.nf;
            for (int c = 0; c < TN; c += 16) {
                uint32_t r[16];
                tmem_ld16(trow + c, r);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int t = t0 + c + j;
                    if (t < a.t) __stcg(wsz + (size_t)t * a.nf + f, __uint_as_float(r[j]));
                }
            }
            __threadfence();
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int tile = blockIdx.y * gridDim.x + blockIdx.x;
            if (threadIdx.x == 64) {
                const int old = atomicAdd(&a.counters[tile], 1);
                s_last = (old == a.splits - 1);
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (s_last) {
                __threadfence();
                const int tend = min(a.t, t0 + TN);
                for (int t = t0; t < tend; ++t) {
                    float acc = __ldcg(a.ws + (size_t)t * a.nf + f);
                    for (int s = 1; s < a.splits; ++s)
                        acc += __ldcg(a.ws + ((size_t)s * a.t + t) * a.nf + f);
                    epi_store<EPI>(a, t, f, acc + bias);
                }
                if (threadIdx.x == 64) a.counters[tile] = 0;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tbase, C::TCOLS);
}

}  // namespace alpa
