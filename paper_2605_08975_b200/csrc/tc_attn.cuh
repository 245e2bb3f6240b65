// tcgen05 dual-source attention for the bf16 path (sm_100a).
//
// emit_attention (model.cpp:280-324) over the attend_view of one block
// (kv_cache.cpp:247-263): every action query of lane l attends the shared
// prefix rows 0..r-1 followed by lane l's own 64 action rows, non-causal,
// scores alpha*dot (alpha applied after the dot, kernels_serial.cpp:24).
//
// One CTA = (head h, query tile of 128 action rows = 2 lanes, KV split s).
// The KV sequence of a tile is the r prefix keys in 128-key blocks, read in
// place from the single prefix copy (TMA, no per-lane replication), plus one
// 128-key "action block" = the two lanes' 64 action keys straight from the QKV
// GEMM output with a block-diagonal lane mask.
//
//   warp 4  TMA producer: Q once; K/V blocks through a 2-stage ring (prefix
//           blocks are prefetched before griddepcontrol.wait: they do not
//           depend on the previous kernel)
//   warp 5  MMA issuer:   S_j = Q.K_j^T into TMEM (double buffered), then
//           O += P_j.V_j (P from smem, V MN-major), S_{j+1} issued before PV_j
//   warps 0-3  softmax:  thread = query row.  tcgen05.ld S row, alpha scale,
//           mask, online max/sum in fp32 (ex2), P row -> bf16 swizzled smem,
//           rescale the TMEM O accumulator when the running max moves.
// KV splits of one tile form a cluster (1,1,S); the partial (O, m, l) of each
// split is merged through DSMEM with the usual log-sum-exp combine.
#pragma once

#include "common.cuh"

namespace alpa {

struct AttnArgs {
    int M;                 // action rows (64 * lanes)
    int r;                 // prefix tokens
    int kv;                // kv width (row stride of ctx, column base of heads)
    int nbp;               // prefix key blocks of 128
    int splits;            // KV splits (= cluster size along z)
    long long pre_k_row;   // row of (block b, K, token 0) in the 2-D prefix view
    long long pre_v_row;   // row of (block b, V, token 0)
    float alpha;           // 1/sqrt(head_dim)
    __nv_bfloat16* ctx;    // [M][kv]
    const void* pf_ptr;    // next op's weights: L2 prefetch, split over the grid
    long long pf_bytes;
};

template <int HD>
struct AttnCfg {
    static constexpr int PANELS = HD / 64;
    static constexpr int Q_BYTES = 128 * HD * 2;
    static constexpr int KV_BYTES = 128 * HD * 2;  // one of K or V for a block
    static constexpr int STAGE = 2 * KV_BYTES;
    static constexpr int P_BYTES = 128 * 128 * 2;
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_KV = Q_BYTES;
    static constexpr int OFF_P = OFF_KV + 2 * STAGE;
    static constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
    static constexpr int SMEM = OFF_BAR + 1536 + 1024;  // barriers + m/l rows + align slack
    static constexpr int O_STRIDE = HD + 4;  // fp32 staging row stride (conflict-free float4)
};

template <int HD>
__global__ void __launch_bounds__(192, 1)
    tc_attn_kernel(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmPre,
                   const AttnArgs a) {
    using C = AttnCfg<HD>;
    extern __shared__ uint8_t smem_raw[];
    // 1024-B aligned (SWIZZLE_128B atoms); offset arithmetic on smem_raw keeps
    // the shared address space visible to the compiler (LDS/STS, not generic)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
    uint64_t* qfull = bars + 0;
    uint64_t* kvfull = bars + 1;   // [2]
    uint64_t* kvempty = bars + 3;  // [2]
    uint64_t* sfull = bars + 5;    // [2]
    uint64_t* sfree = bars + 7;    // [2]
    uint64_t* pfull = bars + 9;    // [2]
    uint64_t* ofull = bars + 11;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
    float* m_sh = reinterpret_cast<float*>(bars + 16);  // [128] (after the barriers)
    float* l_sh = m_sh + 128;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int h = blockIdx.x, qt = blockIdx.y;
    const int S = a.splits;
    const int nb = a.nbp + 1;
    const int g0 = (blockIdx.z * nb) / S, g1 = ((blockIdx.z + 1) * nb) / S;
    const int nj = g1 - g0;
    const int row0 = qt * 128;
    if (threadIdx.x == 0) ALPA_STAMP_AT(0, 0);

    if (threadIdx.x == 0) {
        tma_prefetch(&tmQKV);
        tma_prefetch(&tmPre);
        mbar_init(qfull, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&kvfull[i], 1);
            mbar_init(&kvempty[i], 1);
            mbar_init(&sfull[i], 1);
            mbar_init(&sfree[i], 128);
            mbar_init(&pfull[i], 128);
        }
        mbar_init(ofull, 1);
        fence_mbar_init();
    }
    if (warp == 5) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    const uint32_t tS[2] = {tbase, tbase + 128};
    const uint32_t tO = tbase + 256;
    if (threadIdx.x == 0) ALPA_STAMP_AT(0, 1);

    if (warp == 4) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            auto load_block = [&](int j, bool prefix_only) {
                const int g = g0 + j, st = j & 1;
                uint8_t* kb = smem + C::OFF_KV + st * C::STAGE;
                uint8_t* vb = kb + C::KV_BYTES;
                if (g < a.nbp) {
                    mbar_expect_tx(&kvfull[st], C::STAGE);
                    for (int p = 0; p < C::PANELS; ++p) {
                        tma_load_2d(kb + p * 16384, &tmPre, &kvfull[st], h * HD + p * 64,
                                    (int)(a.pre_k_row + g * 128));
                        tma_load_2d(vb + p * 16384, &tmPre, &kvfull[st], h * HD + p * 64,
                                    (int)(a.pre_v_row + g * 128));
                    }
                } else if (!prefix_only) {
                    mbar_expect_tx(&kvfull[st], C::STAGE);
                    for (int p = 0; p < C::PANELS; ++p) {
                        tma_load_2d(kb + p * 16384, &tmQKV, &kvfull[st], a.kv + h * HD + p * 64, row0);
                        tma_load_2d(vb + p * 16384, &tmQKV, &kvfull[st], 2 * a.kv + h * HD + p * 64,
                                    row0);
                    }
                }
            };
            if (a.pf_bytes > 0) {
                const long long ncta = (long long)gridDim.x * gridDim.y * gridDim.z;
                const long long cta = blockIdx.x + gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z);
                const long long chunk = ((a.pf_bytes + ncta - 1) / ncta + 15) & ~15ll;
                const long long beg = cta * chunk;
                const long long end = beg + chunk < a.pf_bytes ? beg + chunk : a.pf_bytes;
                for (long long o = beg; o < end; o += 32768) {
                    const long long nbytes = end - o < 32768 ? end - o : 32768;
                    l2_prefetch(reinterpret_cast<const uint8_t*>(a.pf_ptr) + o, (uint32_t)(nbytes & ~15ll));
                }
            }
            const int pre = nj < 2 ? nj : 2;
            bool issued[2] = {false, false};
            for (int j = 0; j < pre; ++j)
                if (g0 + j < a.nbp) { load_block(j, true); issued[j] = true; }
            pdl_wait();
            mbar_expect_tx(qfull, C::Q_BYTES);
            for (int p = 0; p < C::PANELS; ++p)
                tma_load_2d(smem + C::OFF_Q + p * 16384, &tmQKV, qfull, h * HD + p * 64, row0);
            for (int j = 0; j < nj; ++j) {
                if (j < 2) {
                    if (!issued[j]) load_block(j, false);
                } else {
                    mbar_wait(&kvempty[j & 1], ((j >> 1) - 1) & 1);
                    load_block(j, false);
                }
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t idS = idesc_bf16(128, 128);
            constexpr uint32_t idO = idesc_bf16(128, HD, true);
            mbar_wait(qfull, 0);
            ALPA_STAMP_AT(0, 2);
            auto issue_s = [&](int j) {
                const int st = j & 1;
                mbar_wait(&kvfull[st], (j >> 1) & 1);
                mbar_wait(&sfree[st], ((j >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint8_t* kb = smem + C::OFF_KV + st * C::STAGE;
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    const uint64_t da = sdesc_k_sw128(smem + C::OFF_Q + (kk >> 2) * 16384) + 2 * (kk & 3);
                    const uint64_t db = sdesc_k_sw128(kb + (kk >> 2) * 16384) + 2 * (kk & 3);
                    tc_mma_bf16(tS[st], da, db, idS, kk > 0 ? 1u : 0u);
                }
                tc_commit(&sfull[st]);
            };
            auto issue_pv = [&](int j) {
                const int st = j & 1;
                mbar_wait(&pfull[st], (j >> 1) & 1);
                tc_fence_after();
                const uint8_t* pb = smem + C::OFF_P + st * C::P_BYTES;
                const uint8_t* vb = smem + C::OFF_KV + st * C::STAGE + C::KV_BYTES;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {  // 128 keys
                    const uint64_t da = sdesc_k_sw128(pb + (kk >> 2) * 16384) + 2 * (kk & 3);
                    const uint64_t db = sdesc_mn_sw128(vb + kk * 2048, 16384);
                    tc_mma_bf16(tO, da, db, idO, (j > 0 || kk > 0) ? 1u : 0u);
                }
                tc_commit(ofull);
                tc_commit(&kvempty[st]);
            };
            if (nj > 0) issue_s(0);
            for (int j = 0; j < nj; ++j) {
                if (j + 1 < nj) issue_s(j + 1);
                issue_pv(j);
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ softmax (warps 0..3)
        const int i = warp * 32 + lane;           // query row within the tile
        const uint32_t lane_off = uint32_t(warp * 32) << 16;
        const float sl2 = a.alpha * 1.4426950408889634f;
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nj; ++j) {
            const int st = j & 1, g = g0 + j;
            mbar_wait(&sfull[st], (j >> 1) & 1);
            if (i == 0 && j == 0) ALPA_STAMP_AT(0, 3);
            tc_fence_after();
            uint32_t sr[128];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(tS[st] + lane_off + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&sfree[st]);
            // key validity: prefix tail beyond r, action keys of the other lane
            int lo = 0, hi = 128;
            if (g < a.nbp) {
                hi = min(128, a.r - g * 128);
            } else {
                lo = (i >> 6) * 64;
                hi = min(lo + 64, a.M - row0);
            }
            float mx = -INFINITY;
#pragma unroll
            for (int k = 0; k < 128; ++k) {
                const float sv = (k >= lo && k < hi) ? __uint_as_float(sr[k]) * sl2 : -INFINITY;
                sr[k] = __float_as_uint(sv);
                mx = fmaxf(mx, sv);
            }
            const float mn = fmaxf(m, mx);
            const float base = mn == -INFINITY ? 0.f : mn;
            const float corr = (m == mn) ? 1.f : ex2(m - base);
            float rs = 0.f;
            uint8_t* prow = smem + C::OFF_P + st * C::P_BYTES + i * 128;
#pragma unroll
            for (int c = 0; c < 16; ++c) {  // 16 chunks of 8 keys
                float p8[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    p8[e] = ex2(__uint_as_float(sr[c * 8 + e]) - base);
                    rs += p8[e];
                }
                uint4 pk;
                __nv_bfloat162 b0 = __floats2bfloat162_rn(p8[0], p8[1]);
                __nv_bfloat162 b1 = __floats2bfloat162_rn(p8[2], p8[3]);
                __nv_bfloat162 b2 = __floats2bfloat162_rn(p8[4], p8[5]);
                __nv_bfloat162 b3 = __floats2bfloat162_rn(p8[6], p8[7]);
                pk.x = *reinterpret_cast<uint32_t*>(&b0);
                pk.y = *reinterpret_cast<uint32_t*>(&b1);
                pk.z = *reinterpret_cast<uint32_t*>(&b2);
                pk.w = *reinterpret_cast<uint32_t*>(&b3);
                const int panel = c >> 3, ch = c & 7;
                *reinterpret_cast<uint4*>(prow + panel * 16384 + ((ch ^ (i & 7)) << 4)) = pk;
            }
            l = l * corr + rs;
            m = mn;
            fence_proxy_async();
            if (j > 0) {
                // O holds sum_{<j} relative to the old max: rescale before PV_j
                mbar_wait(ofull, (j - 1) & 1);
                tc_fence_after();
                // tcgen05.ld/st are warp-collective (.sync.aligned): the branch
                // must be warp-uniform, lanes with corr == 1 just rewrite O.
                if (__any_sync(0xffffffffu, corr != 1.f)) {
#pragma unroll 1
                    for (int c = 0; c < HD; c += 32) {
                        uint32_t o[32];
                        tmem_ld32(tO + lane_off + c, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
                        tmem_st32(tO + lane_off + c, o);
                    }
                    tmem_st_wait();
                }
            }
            tc_fence_before();
            mbar_arrive(&pfull[st]);
        }
        // final accumulator -> fp32 staging (reuses the K/V ring)
        float* stage = reinterpret_cast<float*>(smem + C::OFF_KV);
        if (nj > 0) {
            mbar_wait(ofull, (nj - 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < HD; c += 32) {
                uint32_t o[32];
                tmem_ld32(tO + lane_off + c, o);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; e += 4)
                    *reinterpret_cast<float4*>(stage + i * C::O_STRIDE + c + e) =
                        make_float4(__uint_as_float(o[e]), __uint_as_float(o[e + 1]),
                                    __uint_as_float(o[e + 2]), __uint_as_float(o[e + 3]));
            }
        } else {
            for (int c = 0; c < HD; c += 4)
                *reinterpret_cast<float4*>(stage + i * C::O_STRIDE + c) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (i == 0) ALPA_STAMP_AT(0, 4);
        m_sh[i] = m;  // log2 domain (alpha*log2e folded in)
        l_sh[i] = l;
    }
    tc_fence_before();
    __syncthreads();
    pdl_launch();
    // ------------------------------------------------ split combine + store (all warps)
    // CTA `rank` of the cluster owns rows [rank*128/S, (rank+1)*128/S).  Phase
    // 1 gathers every split's (m, l) for those rows (independent DSMEM loads),
    // phase 2 turns them into per-split weights w_s / L in local smem, phase 3
    // streams the O partials with all S loads of an item in flight.
    {
        const uint32_t rank = S > 1 ? cluster_ctarank() : 0;
        if (S > 1) cluster_sync_all();
        ALPA_STAMP_AT(0, 5);
        const int r_begin = (int)(rank * 128) / S, r_end = (int)((rank + 1) * 128) / S;
        const int rows = r_end - r_begin;
        const uint32_t st_local = smem_u32(smem + C::OFF_KV);
        const uint32_t m_local = smem_u32(m_sh), l_local = smem_u32(l_sh);
        float* wgt = reinterpret_cast<float*>(smem + C::OFF_P);  // [S][rows] (P ring is free)
        float* gm = wgt + 8 * 128;                                // [S][rows] gathered m
        float* gl = gm + 8 * 128;                                 // [S][rows] gathered l
        for (int t = threadIdx.x; t < S * rows; t += 192) {
            const int s2 = t / rows, rr = r_begin + t % rows;
            float mv, lv;
            const uint32_t ma = (S > 1 ? dsmem_addr(m_local, s2) : m_local) + rr * 4;
            const uint32_t la = (S > 1 ? dsmem_addr(l_local, s2) : l_local) + rr * 4;
            asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(mv) : "r"(ma) : "memory");
            asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(lv) : "r"(la) : "memory");
            gm[t] = mv;
            gl[t] = lv;
        }
        __syncthreads();
        for (int rl = threadIdx.x; rl < rows; rl += 192) {
            float M = -INFINITY;
            for (int s2 = 0; s2 < S; ++s2) M = fmaxf(M, gm[s2 * rows + rl]);
            float L = 0.f;
            for (int s2 = 0; s2 < S; ++s2) {
                const float mv = gm[s2 * rows + rl];
                const float w = mv == -INFINITY ? 0.f : ex2(mv - M);
                wgt[s2 * rows + rl] = w;
                L += w * gl[s2 * rows + rl];
            }
            const float inv = 1.0f / L;
            for (int s2 = 0; s2 < S; ++s2) wgt[s2 * rows + rl] *= inv;
        }
        __syncthreads();
        constexpr int CG = HD / 4;  // float4 column groups per row
        uint32_t base[8];
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) base[s2] = (s2 < S && S > 1) ? dsmem_addr(st_local, s2) : st_local;
        for (int it = threadIdx.x; it < rows * CG; it += 192) {
            const int rl = it / CG, cq = (it % CG) * 4;
            const int rr = r_begin + rl;
            const uint32_t off = (uint32_t)(rr * C::O_STRIDE + cq) * 4u;
            float4 p[8];
#pragma unroll
            for (int s2 = 0; s2 < 8; ++s2)
                if (s2 < S) p[s2] = ld_dsmem_f4(base[s2] + off);
            float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int s2 = 0; s2 < 8; ++s2)
                if (s2 < S) {
                    const float w = wgt[s2 * rows + rl];
                    o.x += w * p[s2].x; o.y += w * p[s2].y; o.z += w * p[s2].z; o.w += w * p[s2].w;
                }
            const int t = row0 + rr;
            if (t < a.M) {
                __nv_bfloat162 lo2 = __floats2bfloat162_rn(o.x, o.y);
                __nv_bfloat162 hi2 = __floats2bfloat162_rn(o.z, o.w);
                uint2 pk;
                pk.x = *reinterpret_cast<uint32_t*>(&lo2);
                pk.y = *reinterpret_cast<uint32_t*>(&hi2);
                *reinterpret_cast<uint2*>(a.ctx + (int64_t)t * a.kv + blockIdx.x * HD + cq) = pk;
            }
        }
        ALPA_STAMP_AT(0, 6);
        if (S > 1) cluster_sync_all();
    }
    if (warp == 5) tmem_dealloc(tbase, 512);
    if (threadIdx.x == 160) ALPA_STAMP_AT(0, 7);
}

}  // namespace alpa
