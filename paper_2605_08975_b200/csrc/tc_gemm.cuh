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
// Epilogue: the accumulator is staged TMEM -> registers -> smem (fp32
// [token][feature], reusing the drained pipeline buffers), then ALL 192
// threads apply bias / GELU / residual with coalesced 16-byte global
// accesses along the feature dimension.
//
// Split-K is deterministic and on-chip: the S CTAs that share an output tile
// form one thread-block cluster (1,1,S).  CTA s owns token rows
// [s*TN/S, (s+1)*TN/S): after staging, every CTA pushes each other owner's row
// slice into that owner's receive slots with one TMA bulk copy
// (smem -> DSMEM, completing on the owner's mbarrier); the owner then sums the
// S slices from LOCAL smem in split order and applies the fused epilogue.
#pragma once

#include "common.cuh"

namespace alpa {

enum Epi : int {
    EPI_BF16 = 0,       // out bf16 = acc + b                      (QKV, model.cpp:574-576)
    EPI_GELU_BF16 = 1,  // out bf16 = gelu(acc + b)                (mlp1 + gelu, model.cpp:585-586)
    EPI_F32 = 2,        // out f32  = acc + b                      (encoder mlp2, model.cpp:562)
    EPI_RESID_F32 = 3,  // out f32  = out + (acc + b)              (o / mlp2 + residual, model.cpp:582-588)
    EPI_NONE = 4,       // benchmarking only: accumulator discarded
    EPI_LN_BF16 = 5,    // out bf16 = rstd*(acc - mu*colsum) + b   (LN1 folded into QKV)
    EPI_LN_GELU_BF16 = 6,  // out bf16 = gelu(rstd*(acc - mu*colsum) + b)  (LN2 folded into mlp1)
};
// LayerNorm fold (gamma = 1, beta = 0, model.cpp:83-88): with x = bf16(e),
//   LN(e).W = rstd * (x.W - mu * colsum(W)),  colsum(W)[f] = sum_k W[f][k].
// The residual-producing GEMMs (EPI_F32 / EPI_RESID_F32) emit, next to the
// fp32 stream e, its bf16 copy and per-(row, 128-feature tile) partial
// (sum, sum of squares); the consumer reduces the tile partials of its rows in
// a fixed order (deterministic) to mu and rstd = 1/sqrt(var + 1e-5).

struct GemmArgs {
    int nf, t, k;          // features (MMA M), tokens (MMA N), reduction
    const float* bias;     // [nf]
    void* out;             // [t][ldo]
    int64_t ldo;
    int splits, kbs;       // split-K count (= cluster size along z), k-blocks per split
    // LN fold side channels
    float2* stats_out;             // [t][nft] (sum, sumsq) of the new e rows, or null
    __nv_bfloat16* xb_out;         // [t][nf]  bf16 copy of the new e rows, or null
    const float2* stats_in;        // [t][nft] partials of the LN input rows
    const float* colsum;           // [nf] column sums of the bf16 weights
    int nft;                       // feature tiles per stats row
    int ln_n;                      // LayerNorm width
    int trace;                     // debug builds: stamp this launch's phases
    const void* pf_ptr;            // next op's weights: L2 prefetch, split over the grid
    long long pf_bytes;
};

template <int TN>
struct GemmCfg {
    static constexpr int W_BYTES = 128 * 64 * 2;
    static constexpr int X_BYTES = TN * 64 * 2;
    static constexpr int STAGE = W_BYTES + X_BYTES;
#ifdef ALPA_GEMM_STAGES
    static constexpr int STAGES = ALPA_GEMM_STAGES;
#else
    static constexpr int STAGES = (200 * 1024) / STAGE > 8 ? 8 : (200 * 1024) / STAGE;
#endif
    static constexpr int TAIL = 256 + 8 * 256;  // barriers + tmem slot + LN row stats
    static constexpr int SMEM = STAGES * STAGE + 1024 + TAIL;
    static constexpr uint32_t TCOLS = TN <= 32 ? 32 : TN <= 64 ? 64 : TN <= 128 ? 128 : 256;
    static constexpr int THREADS = 320;         // TMA, MMA, 8 epilogue warps
    static constexpr int NW = THREADS / 32;
};

// 4 consecutive features of one token row: v = acc + bias, then the op.
template <int EPI>
__device__ inline void epi_store4(const GemmArgs& a, int t, int f, float4 v) {
    if constexpr (EPI == EPI_BF16 || EPI == EPI_GELU_BF16) {
        if constexpr (EPI == EPI_GELU_BF16) {
            v.x = gelu_fast(v.x); v.y = gelu_fast(v.y); v.z = gelu_fast(v.z); v.w = gelu_fast(v.w);
        }
        __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(a.out) + (int64_t)t * a.ldo + f) = pk;
    } else if constexpr (EPI == EPI_F32) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + (int64_t)t * a.ldo + f) = v;
    } else if constexpr (EPI == EPI_RESID_F32) {
        float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + (int64_t)t * a.ldo + f);
        const float4 e = *o;
        *o = make_float4(e.x + v.x, e.y + v.y, e.z + v.z, e.w + v.w);
    }
}

template <int TN, int EPI>
__global__ void __launch_bounds__(320, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const GemmArgs a) {
    using C = GemmCfg<TN>;
    constexpr bool LN_IN = (EPI == EPI_LN_BF16 || EPI == EPI_LN_GELU_BF16);
    extern __shared__ uint8_t smem_raw[];
    // 1024-B aligned (SWIZZLE_128B atoms); offset arithmetic on smem_raw keeps
    // the shared address space visible to the compiler (LDS/STS, not generic)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
    uint64_t* empty = full + C::STAGES;
    uint64_t* accf = empty + C::STAGES;
    uint64_t* recvb = accf + 1;  // split-K receive barrier
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recvb + 1);
    float* mu_s = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE + 256);  // [TN]
    float* rs_s = mu_s + 256;                                                   // [TN]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int f0 = blockIdx.x * 128, t0 = blockIdx.y * TN;
    const int KB = a.k / 64;
    const int kb0 = blockIdx.z * a.kbs;
    const int nkb = min(KB, kb0 + a.kbs) - kb0;
    if (threadIdx.x == 0) if (a.trace) ALPA_STAMP_AT(2048, 0);

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmW);
        tma_prefetch(&tmX);
        for (int i = 0; i < C::STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(accf, 1);
        mbar_init(recvb, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, C::TCOLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    if (threadIdx.x == 0) if (a.trace) ALPA_STAMP_AT(2048, 1);

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
                if (i == pre - 1) {
                    // this CTA's share of the NEXT op's weights -> L2 (HBM streams
                    // while this op computes, the epilogue and the launch gap)
                    if (a.pf_bytes > 0) {
                        const long long ncta = (long long)gridDim.x * gridDim.y * gridDim.z;
                        const long long cta = blockIdx.x + gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z);
                        const long long chunk = ((a.pf_bytes + ncta - 1) / ncta + 15) & ~15ll;
                        const long long beg = cta * chunk;
                        const long long end = beg + chunk < a.pf_bytes ? beg + chunk : a.pf_bytes;
                        for (long long o = beg; o < end; o += 32768) {
                            const long long n = end - o < 32768 ? end - o : 32768;
                            l2_prefetch(reinterpret_cast<const uint8_t*>(a.pf_ptr) + o, (uint32_t)(n & ~15ll));
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16(128, TN);
            for (int i = 0; i < nkb; ++i) {
                const int st = i % C::STAGES;
                const uint32_t ph = (i / C::STAGES) & 1;
                mbar_wait(&full[st], ph);
                if (i == 0) if (a.trace) ALPA_STAMP_AT(2048, 2);
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
        // ---------------- epilogue warps 2..9 ---------------------------------
        // While the mainloop runs: LayerNorm statistics of this tile's token
        // rows from the producer's per-tile partials (fixed reduction order).
        if constexpr (LN_IN) {
            pdl_wait();
            const int et = threadIdx.x - 64;  // 0..255
            if (et < TN) {
                const int t = t0 + et;
                float s1 = 0.f, s2 = 0.f;
                if (t < a.t) {
                    const float2* p = a.stats_in + (int64_t)t * a.nft;
                    for (int j = 0; j < a.nft; ++j) {
                        const float2 v = p[j];
                        s1 += v.x;
                        s2 += v.y;
                    }
                }
                const float inv_n = 1.0f / (float)a.ln_n;
                const float mu = s1 * inv_n;
                const float var = fmaxf(s2 * inv_n - mu * mu, 0.f);
                mu_s[et] = mu;
                rs_s[et] = 1.0f / sqrtf(var + 1e-5f);
            }
        }
        // stage 1: TMEM -> smem [token][feature] fp32; 2 warps per lane quarter,
        // each taking half of the token columns
        const int q = warp & 3, half = (warp - 2) >> 2;
        const uint32_t trow = tbase + (uint32_t(q * 32) << 16);
        float* stage = reinterpret_cast<float*>(smem);  // [TN][128] fp32
        mbar_wait(accf, 0);
        if (threadIdx.x == 64) if (a.trace) ALPA_STAMP_AT(2048, 3);
        tc_fence_after();
        const int fl = q * 32 + lane;
        constexpr int HALF = TN / 2;
#pragma unroll 1
        for (int c = half * HALF; c < (half + 1) * HALF; c += 16) {
            uint32_t r[16];
            tmem_ld16(trow + c, r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) stage[(c + j) * 128 + fl] = __uint_as_float(r[j]);
        }
    }
    tc_fence_before();
    __syncthreads();
    pdl_launch();
    // ---------------- epilogue stage 2: reduce + fused op (all 10 warps) -------
    {
        const int S = a.splits;
        const int rows = TN / S;
        const uint32_t rank = S > 1 ? cluster_ctarank() : 0;
        float* stage = reinterpret_cast<float*>(smem);
        float* recv = stage + TN * 128;  // (S-1) slots of [rows][128]
        const uint32_t slice_bytes = (uint32_t)rows * 512u;
        if (S > 1 && threadIdx.x == 0) mbar_expect_tx(recvb, (uint32_t)(S - 1) * slice_bytes);
        if (threadIdx.x == 0) if (a.trace) ALPA_STAMP_AT(2048, 4);
        if (S > 1) cluster_sync_all();  // every split staged; receive slots are free
        if (threadIdx.x == 0) if (a.trace) ALPA_STAMP_AT(2048, 5);
        if (S > 1) {
            if (threadIdx.x == 0) {
                const uint32_t recv_local = smem_u32(recv), bar_local = smem_u32(recvb);
                for (int d = 0; d < S; ++d) {
                    if (d == (int)rank) continue;
                    const int slot = (int)rank < d ? (int)rank : (int)rank - 1;
                    bulk_copy_to_cluster(dsmem_addr(recv_local + slot * slice_bytes, d),
                                         smem_u32(stage + d * rows * 128), slice_bytes,
                                         dsmem_addr(bar_local, d));
                }
            }
            mbar_wait(recvb, 0);
        }
        const int r0 = (int)rank * rows;
        const int fq = lane * 4;  // 4 features per lane
        const float4 b4 = *reinterpret_cast<const float4*>(a.bias + f0 + fq);
        pdl_wait();  // residual / outputs may be touched by the previous kernel
        float4 c4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if constexpr (LN_IN) c4 = *reinterpret_cast<const float4*>(a.colsum + f0 + fq);
        constexpr int NW = C::NW;
        // 4 rows per warp pass, every load of the pass in flight at once
        for (int rb = warp; rb < rows; rb += 4 * NW) {
            float4 acc[4];
            float4 res[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int rl = rb + NW * u;
                const int tl = r0 + rl;
                acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                res[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (rl >= rows) continue;
                if (S > 1) {
                    // fixed split order 0..S-1: own slice from staging, others from slots
                    for (int s2 = 0; s2 < S; ++s2) {
                        const float* src = s2 == (int)rank
                                               ? stage + tl * 128
                                               : recv + ((s2 < (int)rank ? s2 : s2 - 1) * rows + rl) * 128;
                        const float4 p = *reinterpret_cast<const float4*>(src + fq);
                        acc[u].x += p.x; acc[u].y += p.y; acc[u].z += p.z; acc[u].w += p.w;
                    }
                } else {
                    acc[u] = *reinterpret_cast<const float4*>(stage + tl * 128 + fq);
                }
                const int t = t0 + tl;
                if constexpr (EPI == EPI_RESID_F32)
                    if (t < a.t)
                        res[u] = *reinterpret_cast<const float4*>(
                            reinterpret_cast<const float*>(a.out) + (int64_t)t * a.ldo + f0 + fq);
            }
            float4 v[4];
            bool ok[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int rl = rb + NW * u;
                const int tl = r0 + rl;
                ok[u] = rl < rows && t0 + tl < a.t;  // warp-uniform
                v[u] = make_float4(acc[u].x + b4.x, acc[u].y + b4.y, acc[u].z + b4.z, acc[u].w + b4.w);
                if constexpr (LN_IN) {
                    const float mu = ok[u] ? mu_s[tl] : 0.f, rstd = ok[u] ? rs_s[tl] : 0.f;
                    v[u] = make_float4(rstd * (acc[u].x - mu * c4.x) + b4.x,
                                       rstd * (acc[u].y - mu * c4.y) + b4.y,
                                       rstd * (acc[u].z - mu * c4.z) + b4.z,
                                       rstd * (acc[u].w - mu * c4.w) + b4.w);
                }
                if constexpr (EPI == EPI_RESID_F32)
                    v[u] = make_float4(res[u].x + v[u].x, res[u].y + v[u].y, res[u].z + v[u].z,
                                       res[u].w + v[u].w);
            }
            if constexpr (EPI == EPI_RESID_F32 || EPI == EPI_F32) {
                float ps[4], pq[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    ps[u] = v[u].x + v[u].y + v[u].z + v[u].w;
                    pq[u] = v[u].x * v[u].x + v[u].y * v[u].y + v[u].z * v[u].z + v[u].w * v[u].w;
                }
                if (a.stats_out) {
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            ps[u] += __shfl_xor_sync(0xffffffffu, ps[u], o);
                            pq[u] += __shfl_xor_sync(0xffffffffu, pq[u], o);
                        }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (!ok[u]) continue;
                    const int t = t0 + r0 + rb + NW * u;
                    *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + (int64_t)t * a.ldo +
                                               f0 + fq) = v[u];
                    if (a.stats_out) {
                        if (lane == 0)
                            a.stats_out[(int64_t)t * a.nft + blockIdx.x] = make_float2(ps[u], pq[u]);
                        __nv_bfloat162 lo = __floats2bfloat162_rn(v[u].x, v[u].y);
                        __nv_bfloat162 hi = __floats2bfloat162_rn(v[u].z, v[u].w);
                        uint2 pk;
                        pk.x = *reinterpret_cast<uint32_t*>(&lo);
                        pk.y = *reinterpret_cast<uint32_t*>(&hi);
                        *reinterpret_cast<uint2*>(a.xb_out + (int64_t)t * a.ldo + f0 + fq) = pk;
                    }
                }
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (!ok[u]) continue;
                    const int t = t0 + r0 + rb + NW * u;
                    if constexpr (EPI == EPI_LN_BF16) epi_store4<EPI_BF16>(a, t, f0 + fq, v[u]);
                    else if constexpr (EPI == EPI_LN_GELU_BF16) epi_store4<EPI_GELU_BF16>(a, t, f0 + fq, v[u]);
                    else epi_store4<EPI>(a, t, f0 + fq, v[u]);
                }
            }
        }
        if (threadIdx.x == 0) if (a.trace) ALPA_STAMP_AT(2048, 6);
        if (S > 1) cluster_sync_all();  // keep smem alive until every CTA read it
    }
    if (warp == 1) tmem_dealloc(tbase, C::TCOLS);
    if (threadIdx.x == 32) if (a.trace) ALPA_STAMP_AT(2048, 7);
}

}  // namespace alpa
