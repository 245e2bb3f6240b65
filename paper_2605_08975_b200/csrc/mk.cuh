// Persistent denoising-iteration kernel for the bf16 tensor-core path (sm_100a).
//
// ONE launch runs a whole diffusion iteration (Model::run_action_iteration,
// model.cpp:600-605): encode, encoder MLP, every decoder block (QKV with LN1
// folded, attention over [shared prefix || own action block], O + residual,
// MLP1 with LN2 folded + GELU, MLP2 + residual) and LN_f + head + Euler update.
// One CTA per SM stays resident for the whole iteration; the op sequence is a
// device-side plan (Op[]), every CTA walks it in the same order and takes the
// items i = blockIdx.x, blockIdx.x + G, ... of each op.
//
// Why persistent: at N = 6 one op is 4-10 us of tensor work spread over 148
// SMs, and a separate kernel per op pays ~5 us of launch + prologue + pipeline
// fill + drain (measured: tools/gemm_bench, k-block slope vs intercept).  Here
// the TMEM allocation, barrier setup and tensor-map fetches happen once, and
// the TMA producer streams the NEXT item's weights into the smem ring while the
// current item's epilogue drains and while it waits for the op's inputs.
//
// Ordering between ops: a completion counter per op (done[o]), incremented once
// per finished item with release semantics after the item's outputs are
// globally visible (generic stores, then fence.proxy.async so the next op's
// TMA reads see them).  A consumer waits for done[dep] == items(dep) with
// acquire loads.  Every CTA processes ops in plan order and only ever waits on
// earlier ops, so the schedule cannot deadlock with all CTAs co-resident
// (cooperative launch, grid <= #SMs).
//
// Split-K (GEMM) and KV-split (attention) partials go through an fp32
// workspace in L2; the S CTAs of one tile (always one wave, co-resident) meet
// on a per-tile counter and each reduces 1/S of the tile's rows in a FIXED
// split order, so results are deterministic (graph == eager bitwise).
//
// Warp roles (320 threads): warp 0 TMA producer, warp 1 TMEM allocator + MMA
// issuer, warps 2..9 epilogue / softmax / elementwise (256 threads; TMEM lane
// quarter = warp & 3, column half = (warp - 2) >> 2).
#pragma once

#include "common.cuh"
#include "tc_gemm.cuh"

#include <type_traits>

namespace alpa {
namespace mk {

enum OpKind : int { OP_ENCODE = 0, OP_GEMM = 1, OP_ATTN = 2, OP_HEAD = 3 };
enum MkFlags : int { MK_NO_L2PF = 1, MK_NO_PRELOAD = 2, MK_L2_NORMAL = 8 };

struct Op {
    int kind, epi;
    int nf, k;               // GEMM: output features (MMA M side), reduction
    int kbs, splits;         // k-blocks per split, split count (GEMM and attention)
    int tiles_f, tiles_t;    // GEMM tile grid; attention: heads, query tiles
    int n_items;
    int dep, dep_count;      // op whose completion gates this op's inputs, its item count
    int split_base;          // first per-tile split counter of this op
    int nbp;                 // attention: 64-key prefix blocks
    int tn;                  // GEMM: token tile of this op (<= the kernel's TN)
    const CUtensorMap* tmW;  // GEMM: W^T [nf][k] box {64,128}; attention: prefix box {64,64}
    const CUtensorMap* tmX;  // GEMM: X [M][k] box {64,TN};     attention: qkv box {64,64}
    const CUtensorMap* tmQ;  // attention: qkv box {64,128}
    const CUtensorMap* tmO;  // GEMM, unsplit bf16 output: TMA store map, box {64,TN}
    const CUtensorMap* tmXB; // GEMM, unsplit residual producer: bf16 copy map, box {64,TN}
    const CUtensorMap* tmEs; // GEMM, split residual producer: fp32 rows, box {128, TN/S}
    const CUtensorMap* tmXs; // GEMM, split residual producer: bf16 copy, box {64, TN/S}
    const float* bias;
    const float* colsum;     // LN-folded consumers
    void* out;
    long long ldo;
    float2* stats_out;       // residual producers: (sum, sumsq) per (row, 128-feature tile)
    __nv_bfloat16* xb_out;   // residual producers: bf16 copy of the new residual rows
    const float2* stats_in;  // LN consumers
    const void* pf_ptr;      // bytes to pull into L2 while this op runs (a later op's weights)
    long long pf_bytes;
    long long pre_k_row, pre_v_row;  // attention: rows of this block's K / V in the prefix map
};

struct Params {
    const Op* ops;
    int n_ops;
    int* done;        // [n_ops] item completion counters (zeroed before each launch)
    int* splitc;      // per-tile split rendezvous counters
    float* ws;        // split partials (fp32)
    float2* wsml;     // attention (m, l) partials
    int M, ah, kv, H, r, nft;
    float alpha, update_scale;
    float* actions;   // [M][2]
    const float* w_in;
    const float* b_in;
    const float* pos;
    const float* w_head;
    const float* b_head;
    float* e;              // fp32 residual stream [M][ah]
    __nv_bfloat16* x;      // bf16 GEMM operand [M][ah]
    unsigned long long* tstamp;  // optional [n_ops]: completion time per op (profiling)
    int flags;                   // MK_NO_L2PF / MK_NO_PRELOAD (A/B experiments)
    unsigned long long* trace;   // optional [n_ops][G][16]: per-CTA event times (diagnostics)
};

// Trace events (diagnostics build of a launch, p.trace != null).
enum TraceEv : int {
    TR_DEP = 0,      // producer: input dependency satisfied
    TR_MMA0 = 1,     // MMA: first stage of the item landed
    TR_MMA1 = 2,     // MMA: last MMA of the item issued
    TR_ACC = 3,      // epilogue: accumulator ready
    TR_MEET = 4,     // epilogue: split rendezvous passed
    TR_PUB = 5,      // epilogue: item published
    TR_PRE = 6,      // producer: weight prefetch stages issued
    TR_DRAIN = 7,    // epilogue: accumulator drained (stores / partials issued)
    TR_FIX = 8,      // epilogue: fixup done (before the publish fences)
    TR_FENCE = 9,    // epilogue: publish fences + barrier passed
    TR_LOOP = 10,    // epilogue warp 2: drain loop done
    TR_BAR = 11,     // epilogue warp 2: staging barrier passed
    TR_ACC9 = 12,    // epilogue warp 9: accumulator ready
    TR_LOOP9 = 13,   // epilogue warp 9: drain loop done
};

template <int TN, int HD>
struct Cfg {
    static constexpr int W_BYTES = 128 * 64 * 2;
    static constexpr int X_BYTES = TN * 64 * 2;
    static constexpr int KVB = 64 * HD * 2;       // K (or V) of one 64-key block
    static constexpr int KPANEL = 64 * 64 * 2;    // one 64-dim panel of a 64-row tile
    static constexpr int QPANEL = 128 * 64 * 2;   // one 64-dim panel of the 128-row Q tile
    static constexpr int G_SLOT = W_BYTES + X_BYTES;
    static constexpr int A_SLOT = 2 * KVB;
    static constexpr int SLOT = ((G_SLOT > A_SLOT ? G_SLOT : A_SLOT) + 1023) / 1024 * 1024;
    static constexpr int Q_BYTES = 128 * HD * 2;
    static constexpr int P_BYTES = 128 * 64 * 2;  // one 128 x 64 bf16 P tile (one SW128 panel)
    // epilogue staging of a bf16 [TN][128] output tile (two SW128 panels) +
    // scratch (LN mu/rstd, row-stat partials); shares the AUX region with the
    // attention Q and P tiles (ops are sequential within a CTA)
    static constexpr int STG_BYTES = TN * 128 * 2;  // also >= split rows x (512 + 256) B (S >= 4 at TN 192)
    static constexpr int SCR_BYTES = 12 * 1024;
    static constexpr int AUX_ATT = Q_BYTES + 2 * P_BYTES;
    static constexpr int AUX = AUX_ATT > STG_BYTES + SCR_BYTES ? AUX_ATT : STG_BYTES + SCR_BYTES;
    static constexpr int BAR_BYTES = 1024;
    static constexpr int LIMIT = 227 * 1024;
    static constexpr int ST_RAW = (LIMIT - 1024 - AUX - BAR_BYTES) / SLOT;
    static constexpr int STAGES = ST_RAW > 8 ? 8 : ST_RAW;
    static constexpr int OFF_Q = STAGES * SLOT;
    static constexpr int OFF_P = OFF_Q + Q_BYTES;
    static constexpr int OFF_STG = OFF_Q;
    static constexpr int OFF_SCR = OFF_Q + STG_BYTES;
    static constexpr int OFF_BAR = OFF_Q + AUX;
    static constexpr int SMEM = OFF_BAR + BAR_BYTES + 1024;
    static constexpr int THREADS = 320;
    static_assert(STAGES >= 2, "smem ring too small");
    static_assert(SMEM <= LIMIT, "smem budget");
};

// ------------------------------------------------------------------ sync helpers
__device__ inline int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ inline void red_release_add(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ inline void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ inline void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ inline float4 ldcg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
// Explicit global-space stores (op.out is void*: a plain store compiles to a
// generic ST; the global form is the cheaper STG).
__device__ inline void stg(float* p, float v) {
    asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ inline void stg(__nv_bfloat16* p, float v) {
    const __nv_bfloat16 b = __float2bfloat16_rn(v);
    asm volatile("st.global.b16 [%0], %1;" ::"l"(p), "h"(*reinterpret_cast<const unsigned short*>(&b)) : "memory");
}

// Spin until *ctr >= want.  A schedule bug must not hang the GPU: after ~2^24
// polls (seconds) the kernel traps, the launch fails and the host reports it.
// Polls are relaxed (an acquire load invalidates L1 on every poll); one
// acquire load after the count is reached orders the consumer's reads.
__device__ inline int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __noinline__ void wait_count(const int* ctr, int want) {
    uint32_t n = 0;
    while (ld_relaxed(ctr) < want) {
        __nanosleep(64);
        if (++n > (1u << 24)) {
            printf("alpa mk watchdog: block %d thread %d waits counter %p = %d < %d\n", blockIdx.x, threadIdx.x,
                   (const void*)ctr, ld_relaxed(ctr), want);
            __trap();
        }
    }
    (void)ld_acquire(ctr);
}

__device__ inline void stamp(const Params& p, int o) {
    if (p.tstamp) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(p.tstamp + o, t);
    }
}

__device__ inline void trace_ev(const Params& p, int o, int ev) {
    if (p.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[((size_t)o * gridDim.x + blockIdx.x) * 16 + ev] = t;
    }
}

// L2 prefetch of this CTA's 1/G share of a byte range.
__device__ inline void l2_share(const void* ptr, long long bytes, uint64_t pol) {
    if (bytes <= 0) return;
    const long long G = gridDim.x;
    const long long chunk = ((bytes + G - 1) / G + 15) & ~15ll;
    const long long beg = (long long)blockIdx.x * chunk;
    const long long end = beg + chunk < bytes ? beg + chunk : bytes;
    for (long long o = beg; o < end; o += 32768) {
        const long long n = end - o < 32768 ? end - o : 32768;
        if (n >= 16) l2_prefetch_hint(reinterpret_cast<const uint8_t*>(ptr) + o, (uint32_t)(n & ~15ll), pol);
    }
}

struct GemmItem {
    int f0, t0, s, tile, kb0, nkb;
};
__device__ inline GemmItem gemm_item(const Op& op, int it, int TN) {
    GemmItem g;
    g.s = it % op.splits;
    g.tile = it / op.splits;
    g.f0 = (g.tile % op.tiles_f) * 128;
    g.t0 = (g.tile / op.tiles_f) * TN;
    const int KB = op.k / 64;
    g.kb0 = g.s * op.kbs;
    const int e = g.kb0 + op.kbs < KB ? g.kb0 + op.kbs : KB;
    g.nkb = e - g.kb0;
    return g;
}
struct AttnItem {
    int h, qt, s, tile, row0, g0, nj;
};
__device__ inline AttnItem attn_item(const Op& op, int it, int M) {
    AttnItem a;
    a.s = it % op.splits;
    a.tile = it / op.splits;
    a.h = a.tile % op.tiles_f;
    a.qt = a.tile / op.tiles_f;
    a.row0 = a.qt * 128;
    const int lanes = (M - a.row0) / 64 < 2 ? (M - a.row0) / 64 : 2;
    const int nbt = op.nbp + lanes;
    a.g0 = (a.s * nbt) / op.splits;
    a.nj = ((a.s + 1) * nbt) / op.splits - a.g0;
    return a;
}

// ------------------------------------------------------------------ epilogue pieces
// Only 8 warps per SM run these phases, so every loop keeps many independent
// L2 loads in flight (unrolled, predicated) instead of one round trip per value.

// LayerNorm statistics of row t from the producer's per-tile partials, fixed order.
__device__ inline void ln_stats(const Params& p, const float2* st, int t, float& mu, float& rs) {
    float s1 = 0.f, s2 = 0.f;
    const float2* q = st + (int64_t)t * p.nft;
    for (int j0 = 0; j0 < p.nft; j0 += 16) {
        float2 v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = j0 + u < p.nft ? __ldcg(q + j0 + u) : make_float2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            s1 += v[u].x;
            s2 += v[u].y;
        }
    }
    const float inv_n = 1.0f / (float)p.ah;
    mu = s1 * inv_n;
    const float var = fmaxf(s2 * inv_n - mu * mu, 0.f);
    rs = 1.0f / sqrtf(var + 1e-5f);
}

__device__ inline uint2 pack_bf16x4(float4 v) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    return pk;
}

// Merge the 2S attention partials (S KV splits x 2 key halves) of rows
// [rb, re) of one (head, query tile): log-sum-exp weights, fixed order.
template <int HD>
__device__ inline void attn_fixup(const Params& p, const Op& op, const AttnItem& a, int rb, int re,
                                  int ew, int lane) {
    const int np = op.splits;  // one (already half-merged) partial per KV split
    const int d = lane * 4;
    for (int t = rb + ew; t < re; t += 8) {
        float2 ml[6];
        float4 v[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            ml[q] = q < np ? __ldcg(p.wsml + ((int64_t)q * p.M + t) * p.H + a.h) : make_float2(-INFINITY, 0.f);
            v[q] = (q < np && d < HD) ? ldcg4(p.ws + ((int64_t)q * p.M + t) * p.kv + a.h * HD + d)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float mx = -INFINITY;
#pragma unroll
        for (int q = 0; q < 6; ++q) mx = fmaxf(mx, ml[q].x);
        float L = 0.f;
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            const float w = ml[q].x == -INFINITY ? 0.f : ex2(ml[q].x - mx);
            L += w * ml[q].y;
            o.x += w * v[q].x; o.y += w * v[q].y; o.z += w * v[q].z; o.w += w * v[q].w;
        }
        if (d < HD) {
            const float inv = 1.0f / L;
            *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(op.out) + (int64_t)t * p.kv + a.h * HD + d) =
                pack_bf16x4(make_float4(o.x * inv, o.y * inv, o.z * inv, o.w * inv));
        }
    }
}

// bf16 element (row, feature fl of 128) into the [2 panels][TN rows][128 B]
// SW128 staging image of a TMA store box {64, TN}.
template <int TN>
__device__ inline void sts_bf16_t(uint8_t* base, int row, int fl, float v) {
    const int col = fl & 63;
    uint8_t* a = base + (fl >> 6) * (TN * 128) + row * 128 + ((((col >> 3) ^ (row & 7))) << 4) + (col & 7) * 2;
    *reinterpret_cast<__nv_bfloat16*>(a) = __float2bfloat16_rn(v);
}
#define sts_bf16(base, row, fl, v) sts_bf16_t<TN>(base, row, fl, v)

// Generic drain of one thread's accumulator row (feature fl, ncol tokens from
// column c0 of the tile) for every unsplit GEMM epilogue.  ONE out-of-line copy
// serves all ops, so its code stays in the instruction cache across ops (a
// persistent kernel's per-op specialised epilogues were each cold on every use).
// Element math is branch-free; every optional step is a per-group uniform branch.
//   v = rs*(acc - mu*cs) + b   (mu = 0, rs = 1 without LayerNorm: exact)
//   v = e + v                  (staged residual; 0 otherwise)
//   GELU; f32 store; bf16 into the TMA-store staging; row statistics.
struct DrainArgs {
    uint32_t tacc, testage;  // TMEM: accumulator, staged residual (~0: none)
    int ncol, c0, fl, q, lane, gelu;
    float bf, cs;
    const float* mu_s;       // LayerNorm (mu, rstd) per token or null
    const float* rs_s;
    float* erow;             // f32 output at token c0 (stride ldo) or null
    long long ldo;
    uint8_t* stg;            // bf16 staging image or null
    int stg_panel;           // bytes between the two 64-feature panels
    float2* st_part;         // row-stat partials [4][256] or null
    float* part;             // split-K partial row at token c0 (stride ldo): only this
    int dbg;                 // microbenchmarks only: 1 = no TMEM loads
};
template <bool LN, bool GELU, bool RESID, bool F32, bool STG, bool PART>
__device__ __forceinline__ void drain_t(const DrainArgs& a) {
    const int col = a.fl & 63;
    uint8_t* sbase = STG ? a.stg + (a.fl >> 6) * a.stg_panel + (col & 7) * 2 : nullptr;
#pragma unroll 1
    for (int c = 0; c < a.ncol; c += 8) {
        uint32_t r[8], rv[8];
        if (a.dbg & 1) {
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = rv[j] = __float_as_uint((float)(c + j));
        } else {
            tmem_ld8(a.tacc + c, r);
            if constexpr (RESID) tmem_ld8(a.testage + c, rv);
            tmem_ld_wait();
        }
        if constexpr (PART) {
            float* d = a.part + (long long)c * a.ldo;
#pragma unroll
            for (int j = 0; j < 8; ++j) stg(d + j * a.ldo, __uint_as_float(r[j]));
        } else {
            float v[8];
            float mu[8], rs[8];
            if constexpr (LN) {
                *reinterpret_cast<float4*>(mu) = *reinterpret_cast<const float4*>(a.mu_s + a.c0 + c);
                *reinterpret_cast<float4*>(mu + 4) = *reinterpret_cast<const float4*>(a.mu_s + a.c0 + c + 4);
                *reinterpret_cast<float4*>(rs) = *reinterpret_cast<const float4*>(a.rs_s + a.c0 + c);
                *reinterpret_cast<float4*>(rs + 4) = *reinterpret_cast<const float4*>(a.rs_s + a.c0 + c + 4);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float acc = __uint_as_float(r[j]);
                float x = LN ? rs[j] * (acc - mu[j] * a.cs) + a.bf : acc + a.bf;
                if constexpr (RESID) x = __uint_as_float(rv[j]) + x;
                if constexpr (GELU) x = gelu_tanh(x);
                v[j] = x;
            }
            if constexpr (F32) {
                float* d = a.erow + (long long)c * a.ldo;
#pragma unroll
                for (int j = 0; j < 8; ++j) stg(d + j * a.ldo, v[j]);
            }
            if constexpr (STG) {
                if (!(a.dbg & 2)) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int row = a.c0 + c + j;
                        *reinterpret_cast<__nv_bfloat16*>(sbase + row * 128 + ((((col >> 3) ^ (row & 7))) << 4)) =
                            __float2bfloat16_rn(v[j]);
                    }
                }
            }
            if constexpr (F32) {
                if (a.st_part) {
                    // transpose-reduce: 8 token sums over the warp's 32 features;
                    // lane ends with token (lane >> 2) & 7
                    float a1[8], a2[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) { a1[j] = v[j]; a2[j] = v[j] * v[j]; }
#pragma unroll
                    for (int rr = 0; rr < 3; ++rr) {
                        const int off = 16 >> rr, half = 4 >> rr;
                        const bool up = (a.lane & off) != 0;
#pragma unroll
                        for (int i2 = 0; i2 < half; ++i2) {
                            const float s1 = up ? a1[i2] : a1[i2 + half];
                            const float s2 = up ? a2[i2] : a2[i2 + half];
                            const float k1 = up ? a1[i2 + half] : a1[i2];
                            const float k2 = up ? a2[i2 + half] : a2[i2];
                            a1[i2] = k1 + __shfl_xor_sync(0xffffffffu, s1, off);
                            a2[i2] = k2 + __shfl_xor_sync(0xffffffffu, s2, off);
                        }
                    }
                    a1[0] += __shfl_xor_sync(0xffffffffu, a1[0], 2);
                    a2[0] += __shfl_xor_sync(0xffffffffu, a2[0], 2);
                    a1[0] += __shfl_xor_sync(0xffffffffu, a1[0], 1);
                    a2[0] += __shfl_xor_sync(0xffffffffu, a2[0], 1);
                    if ((a.lane & 3) == 0)
                        a.st_part[a.q * 256 + a.c0 + c + ((a.lane >> 2) & 7)] = make_float2(a1[0], a2[0]);
                }
            }
        }
    }
}

// Split-K finalisation of one thread's owned tokens (TMEM layout): the own
// split's partial is read from TMEM, the others' from the L2 workspace, summed
// in split order 0..S-1 (deterministic), + bias (+ staged residual).
struct FixArgs {
    uint32_t tacc, testage;
    int ncol, c0, S, s_own, nf, q, lane;
    const float* ws;          // workspace at (split 0, first owned token, feature)
    long long split_stride;   // floats between splits
    float bf;
    float* erow;              // direct stores (staging does not fit): f32 output at the first owned token
    __nv_bfloat16* xrow;      //   and its bf16 copy (or null)
    long long ldo;
    float* e_stg;             // fp32 staging [rows][128] (TMA store of the e rows), null: direct stores
    uint8_t* x_stg;           // bf16 staging, SW128 panels of [rows][64] (null: no copy)
    int rows;                 // owned rows of the tile (staging row count)
    int r0;                   // this thread's first staging row
    float2* st_part;
};
template <bool RESID>
__device__ __forceinline__ void fix_t(const FixArgs& a) {
#pragma unroll 1
    for (int c = 0; c < a.ncol; c += 8) {
        float pv[4][8];
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2)
#pragma unroll
            for (int j = 0; j < 8; ++j)
                pv[s2][j] = (s2 < a.S && s2 != a.s_own) ? __ldcg(a.ws + s2 * a.split_stride + (long long)(c + j) * a.nf) : 0.f;
        uint32_t r[8], rv[8];
        tmem_ld8(a.tacc + c, r);
        if constexpr (RESID) tmem_ld8(a.testage + c, rv);
        tmem_ld_wait();
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float acc = 0.f;
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2)  // fixed split order 0..S-1
                if (s2 < a.S) acc += (s2 == a.s_own) ? __uint_as_float(r[j]) : pv[s2][j];
            float x = acc + a.bf;
            if constexpr (RESID) x = __uint_as_float(rv[j]) + x;
            v[j] = x;
        }
        const int fl = a.q * 32 + a.lane;
        if (!a.e_stg) {
            float* d = a.erow + (long long)c * a.ldo;
#pragma unroll
            for (int j = 0; j < 8; ++j) stg(d + j * a.ldo, v[j]);
            if (a.xrow) {
#pragma unroll
                for (int j = 0; j < 8; ++j) stg(a.xrow + (long long)(c + j) * a.ldo, v[j]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) a.e_stg[(a.r0 + c + j) * 128 + fl] = v[j];
        }
        if (a.e_stg && a.x_stg) {
            const int col = fl & 63;
            uint8_t* xb = a.x_stg + (fl >> 6) * (a.rows * 128) + (col & 7) * 2;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int row = a.r0 + c + j;
                *reinterpret_cast<__nv_bfloat16*>(xb + row * 128 + ((((col >> 3) ^ (row & 7))) << 4)) =
                    __float2bfloat16_rn(v[j]);
            }
        }
        if (a.st_part) {
            float a1[8], a2[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) { a1[j] = v[j]; a2[j] = v[j] * v[j]; }
#pragma unroll
            for (int rr = 0; rr < 3; ++rr) {
                const int off = 16 >> rr, half = 4 >> rr;
                const bool up = (a.lane & off) != 0;
#pragma unroll
                for (int i2 = 0; i2 < half; ++i2) {
                    const float s1 = up ? a1[i2] : a1[i2 + half];
                    const float s2v = up ? a2[i2] : a2[i2 + half];
                    const float k1 = up ? a1[i2 + half] : a1[i2];
                    const float k2 = up ? a2[i2 + half] : a2[i2];
                    a1[i2] = k1 + __shfl_xor_sync(0xffffffffu, s1, off);
                    a2[i2] = k2 + __shfl_xor_sync(0xffffffffu, s2v, off);
                }
            }
            a1[0] += __shfl_xor_sync(0xffffffffu, a1[0], 2);
            a2[0] += __shfl_xor_sync(0xffffffffu, a2[0], 2);
            a1[0] += __shfl_xor_sync(0xffffffffu, a1[0], 1);
            a2[0] += __shfl_xor_sync(0xffffffffu, a2[0], 1);
            if ((a.lane & 3) == 0) a.st_part[a.q * 256 + a.c0 + c + ((a.lane >> 2) & 7)] = make_float2(a1[0], a2[0]);
        }
    }
}

// Mode dispatch (each op kind has its own straight-line instance).
__device__ inline void drain(const DrainArgs& a, bool ln, bool gelu, bool resid, bool f32, bool part) {
    if (part) drain_t<false, false, false, false, false, true>(a);
    else if (resid) drain_t<false, false, true, true, true, false>(a);
    else if (f32) drain_t<false, false, false, true, true, false>(a);
    else if (ln && gelu) drain_t<true, true, false, false, true, false>(a);
    else if (ln) drain_t<true, false, false, false, true, false>(a);
    else if (gelu) drain_t<false, true, false, false, true, false>(a);
    else drain_t<false, false, false, false, true, false>(a);
}

// Item outputs are complete: make them visible to later generic and TMA
// (async-proxy) readers, then count the item.
__device__ inline void publish(const Params& p, int o, int et) {
    if (et == 0) {
        trace_ev(p, o, TR_FIX);
        bulk_wait_all();  // this item's TMA stores have landed
    }
    fence_proxy_async_global();
    epi_bar();
    if (et == 0) {
        trace_ev(p, o, TR_FENCE);
        red_release_add(p.done + o, 1);  // release is cumulative over the CTA's writes (bar.sync)
        stamp(p, o);
        trace_ev(p, o, TR_PUB);
    }
}

// Split rendezvous: every split of a tile has written its partial.  Thread 0
// also acquires the op's input dependency, so the fixup may read rows other
// CTAs produced (residual stream, LayerNorm statistics).
__device__ inline void split_meet(const Params& p, const Op& op, int o, int* ctr, int et) {
    const int S = op.splits;
    epi_bar();
    if (et == 0) {
        if (op.dep >= 0) wait_count(p.done + op.dep, op.dep_count);
        red_release_add(ctr, 1);
        wait_count(ctr, S);
    }
    epi_bar();
    if (et == 0) trace_ev(p, o, TR_MEET);
}

// ------------------------------------------------------------------ the kernel
template <int TN, int HD>
__global__ void __launch_bounds__(320, 1) iter_kernel(const __grid_constant__ Params p) {
    using C = Cfg<TN, HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
    uint64_t* full = bars;                    // [STAGES]
    uint64_t* empty = bars + 8;               // [STAGES]
    uint64_t* acc_full = bars + 16;
    uint64_t* acc_empty = bars + 17;
    uint64_t* q_full = bars + 18;
    uint64_t* q_empty = bars + 19;
    uint64_t* s_full = bars + 20;             // [2]
    uint64_t* s_free = bars + 22;             // [2]
    uint64_t* p_full = bars + 24;             // [2]
    uint64_t* p_free = bars + 26;             // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 28);
    float* mu_s = reinterpret_cast<float*>(smem + C::OFF_SCR);  // [256] (GEMM items only)
    float* rs_s = mu_s + 256;
    float2* st_part = reinterpret_cast<float2*>(rs_s + 256);  // [4][256] row-stat partials

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        if (p.tstamp) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            atomicMin(p.tstamp + p.n_ops, t);
        }
        for (int i = 0; i < C::STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 1);
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_free[i], 256);
            mbar_init(&p_full[i], 256);
            mbar_init(&p_free[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;

    if (warp == 0) {
        // ================================================= TMA producer
        if (lane == 0) {
            uint32_t ks = 0, natt = 0;
            // weights and the prefix are streamed once per iteration: evict_first
            // keeps them from displacing the kernel's code and the activations in L2
            const uint64_t wpol = (p.flags & MK_L2_NORMAL) ? policy_evict_normal() : policy_evict_first();
            auto slot_acquire = [&](uint32_t kk) -> uint8_t* {
                const uint32_t st = kk % C::STAGES, ph = (kk / C::STAGES) & 1;
                mbar_wait(&empty[st], ph ^ 1);
                return smem + st * C::SLOT;
            };
            for (int o = 0; o < p.n_ops; ++o) {
                const Op op = p.ops[o];  // register copy: stores must not force reloads
                if (op.kind == OP_GEMM) {
                    tma_prefetch(op.tmW);
                    tma_prefetch(op.tmX);
                    bool waited = false;
                    for (int it = blockIdx.x; it < op.n_items; it += gridDim.x) {
                        const GemmItem g = gemm_item(op, it, op.tn);
                        const uint32_t stage_tx = C::W_BYTES + op.tn * 128;
                        // weights do not depend on earlier ops: start them first
                        int pre = g.nkb < C::STAGES ? g.nkb : C::STAGES;
                        if (p.flags & MK_NO_PRELOAD) {
                            pre = 0;
                            if (!waited && op.dep >= 0) {
                                wait_count(p.done + op.dep, op.dep_count);
                                fence_proxy_async_global();
                                waited = true;
                            }
                        }
                        for (int i = 0; i < pre; ++i) {
                            const uint32_t st = (ks + i) % C::STAGES;
                            uint8_t* sb = slot_acquire(ks + i);
                            mbar_expect_tx(&full[st], stage_tx);
                            tma_load_2d_hint(sb, op.tmW, &full[st], (g.kb0 + i) * 64, g.f0, wpol);
                        }
                        trace_ev(p, o, TR_PRE);
                        if (!waited && op.dep >= 0) {
                            wait_count(p.done + op.dep, op.dep_count);
                            fence_proxy_async_global();
                            waited = true;
                        }
                        trace_ev(p, o, TR_DEP);
                        for (int i = 0; i < g.nkb; ++i) {
                            const uint32_t st = (ks + i) % C::STAGES;
                            uint8_t* sb = smem + st * C::SLOT;
                            if (i >= pre) {
                                sb = slot_acquire(ks + i);
                                mbar_expect_tx(&full[st], stage_tx);
                                tma_load_2d_hint(sb, op.tmW, &full[st], (g.kb0 + i) * 64, g.f0, wpol);
                            }
                            tma_load_2d(sb + C::W_BYTES, op.tmX, &full[st], (g.kb0 + i) * 64, g.t0);
                        }
                        ks += g.nkb;
                    }
                    if (!(p.flags & MK_NO_L2PF)) l2_share(op.pf_ptr, op.pf_bytes, wpol);
                } else if (op.kind == OP_ATTN) {
                    tma_prefetch(op.tmW);
                    tma_prefetch(op.tmX);
                    tma_prefetch(op.tmQ);
                    bool waited = false;
                    for (int it = blockIdx.x; it < op.n_items; it += gridDim.x) {
                        const AttnItem a = attn_item(op, it, p.M);
                        auto load_block = [&](int j) {
                            const uint32_t st = (ks + j) % C::STAGES;
                            uint8_t* kb = slot_acquire(ks + j);
                            uint8_t* vb = kb + C::KVB;
                            mbar_expect_tx(&full[st], 2 * C::KVB);
                            const int gb = a.g0 + j;
                            for (int pn = 0; pn < HD / 64; ++pn) {
                                const int col = a.h * HD + pn * 64;
                                if (gb < op.nbp) {
                                    tma_load_2d_hint(kb + pn * C::KPANEL, op.tmW, &full[st], col,
                                                     (int)(op.pre_k_row + gb * 64), wpol);
                                    tma_load_2d_hint(vb + pn * C::KPANEL, op.tmW, &full[st], col,
                                                     (int)(op.pre_v_row + gb * 64), wpol);
                                } else {
                                    const int row = a.row0 + (gb - op.nbp) * 64;
                                    tma_load_2d(kb + pn * C::KPANEL, op.tmX, &full[st], p.kv + col, row);
                                    tma_load_2d(vb + pn * C::KPANEL, op.tmX, &full[st], 2 * p.kv + col, row);
                                }
                            }
                        };
                        int pre = 0;
                        while (pre < a.nj && pre < C::STAGES && a.g0 + pre < op.nbp) load_block(pre++);
                        trace_ev(p, o, TR_PRE);
                        if (!waited && op.dep >= 0) {
                            wait_count(p.done + op.dep, op.dep_count);
                            fence_proxy_async_global();
                            waited = true;
                        }
                        trace_ev(p, o, TR_DEP);
                        if (natt > 0) mbar_wait(q_empty, (natt - 1) & 1);
                        mbar_expect_tx(q_full, C::Q_BYTES);
                        for (int pn = 0; pn < HD / 64; ++pn)
                            tma_load_2d(smem + C::OFF_Q + pn * C::QPANEL, op.tmQ, q_full,
                                        a.h * HD + pn * 64, a.row0);
                        for (int j = pre; j < a.nj; ++j) load_block(j);
                        ks += a.nj;
                        ++natt;
                    }
                    if (!(p.flags & MK_NO_L2PF)) l2_share(op.pf_ptr, op.pf_bytes, wpol);
                }
            }
        }
    } else if (warp == 1) {
        // ================================================= MMA issuer
        if (lane == 0) {
            uint32_t ks = 0, nmma = 0, natt = 0, J = 0;
            const uint32_t tS[2] = {tbase, tbase + 64};
            const uint32_t tO[2] = {tbase + 128, tbase + 128 + HD};
            for (int o = 0; o < p.n_ops; ++o) {
                const Op op = p.ops[o];  // register copy: stores must not force reloads
                if (op.kind == OP_GEMM) {
                    const uint32_t idesc = idesc_bf16(128, op.tn);
                    for (int it = blockIdx.x; it < op.n_items; it += gridDim.x) {
                        const GemmItem g = gemm_item(op, it, op.tn);
                        if (nmma > 0) mbar_wait(acc_empty, (nmma - 1) & 1);
                        for (int i = 0; i < g.nkb; ++i) {
                            const uint32_t st = (ks + i) % C::STAGES, ph = ((ks + i) / C::STAGES) & 1;
                            mbar_wait(&full[st], ph);
                            if (i == 0) trace_ev(p, o, TR_MMA0);
                            tc_fence_after();
                            uint8_t* sb = smem + st * C::SLOT;
                            const uint64_t da = sdesc_k_sw128(sb);
                            const uint64_t db = sdesc_k_sw128(sb + C::W_BYTES);
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                tc_mma_bf16(tbase, da + 2 * k, db + 2 * k, idesc, (i | k) != 0 ? 1u : 0u);
                            tc_commit(&empty[st]);
                        }
                        tc_commit(acc_full);
                        trace_ev(p, o, TR_MMA1);
                        ks += g.nkb;
                        ++nmma;
                    }
                } else if (op.kind == OP_ATTN) {
                    constexpr uint32_t idS = idesc_bf16(128, 64);
                    constexpr uint32_t idO = idesc_bf16(128, HD, true);
                    for (int it = blockIdx.x; it < op.n_items; it += gridDim.x) {
                        const AttnItem a = attn_item(op, it, p.M);
                        if (nmma > 0) mbar_wait(acc_empty, (nmma - 1) & 1);
                        mbar_wait(q_full, natt & 1);
                        tc_fence_after();
                        auto issue_pv = [&](uint32_t JJ, uint32_t st, bool first) {
                            mbar_wait(&p_full[JJ & 1], (JJ >> 1) & 1);
                            tc_fence_after();
                            const uint8_t* pb = smem + C::OFF_P + (JJ & 1) * C::P_BYTES;
                            const uint8_t* vb = smem + st * C::SLOT + C::KVB;
#pragma unroll
                            for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                                for (int kk = 0; kk < 2; ++kk) {
                                    const int ks16 = hh * 2 + kk;  // 16-key step within the block
                                    const uint64_t da = sdesc_k_sw128(pb) + 2 * ks16;
                                    const uint64_t dbv = sdesc_mn_sw128(vb + ks16 * 2048, C::KPANEL);
                                    tc_mma_bf16(tO[hh], da, dbv, idO, (first && kk == 0) ? 0u : 1u);
                                }
                            tc_commit(&empty[st]);
                            tc_commit(&p_free[JJ & 1]);
                        };
                        uint32_t prev_st = 0;
                        for (int j = 0; j < a.nj; ++j) {
                            const uint32_t JJ = J + j;
                            const uint32_t st = (ks + j) % C::STAGES, ph = ((ks + j) / C::STAGES) & 1;
                            mbar_wait(&full[st], ph);
                            if (j == 0) trace_ev(p, o, TR_MMA0);
                            if (JJ >= 2) mbar_wait(&s_free[JJ & 1], ((JJ - 2) >> 1) & 1);
                            tc_fence_after();
                            const uint8_t* kb = smem + st * C::SLOT;
#pragma unroll
                            for (int kk = 0; kk < HD / 16; ++kk) {
                                const uint64_t da = sdesc_k_sw128(smem + C::OFF_Q + (kk >> 2) * C::QPANEL) + 2 * (kk & 3);
                                const uint64_t db = sdesc_k_sw128(kb + (kk >> 2) * C::KPANEL) + 2 * (kk & 3);
                                tc_mma_bf16(tS[JJ & 1], da, db, idS, kk > 0 ? 1u : 0u);
                            }
                            tc_commit(&s_full[JJ & 1]);
                            if (j == a.nj - 1) tc_commit(q_empty);
                            if (j > 0) issue_pv(JJ - 1, prev_st, j == 1);
                            prev_st = st;
                        }
                        if (a.nj > 0) issue_pv(J + a.nj - 1, prev_st, a.nj == 1);
                        else tc_commit(q_empty);
                        tc_commit(acc_full);
                        trace_ev(p, o, TR_MMA1);
                        ks += a.nj;
                        J += a.nj;
                        ++natt;
                        ++nmma;
                    }
                }
            }
        }
        __syncwarp();
    } else {
        // ================================================= epilogue / softmax / elementwise
        const int et = threadIdx.x - 64;   // 0..255
        const int ew = warp - 2;           // 0..7
        const int q = warp & 3;            // TMEM lane quarter
        const int hh = ew >> 2;            // column half
        const uint32_t lane_off = uint32_t(q * 32) << 16;
        uint32_t nmma = 0, J = 0;
        for (int o = 0; o < p.n_ops; ++o) {
            const Op op = p.ops[o];  // register copy: stores must not force reloads
            if (op.kind == OP_ENCODE) {
                // e0 = a.W_in + b_in + pos (model.cpp:558-559), reference rounding order;
                // thread = 4 consecutive features, all loads of a pass in flight
                for (int it = blockIdx.x; it < op.n_items; it += gridDim.x) {
                    const int r0 = it * 8, r1 = min(p.M, r0 + 8);
                    const int groups = (r1 - r0) * (p.ah / 4);
                    for (int gi0 = et; gi0 < groups; gi0 += 4 * 256) {
                        float4 w0[4], w1[4], bb[4], ps[4];
                        float2 av[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int gi = gi0 + u * 256;
                            if (gi >= groups) continue;
                            const int t = r0 + gi / (p.ah / 4), j = (gi % (p.ah / 4)) * 4;
                            w0[u] = *reinterpret_cast<const float4*>(p.w_in + j);
                            w1[u] = *reinterpret_cast<const float4*>(p.w_in + p.ah + j);
                            bb[u] = *reinterpret_cast<const float4*>(p.b_in + j);
                            ps[u] = *reinterpret_cast<const float4*>(p.pos + (t % 64) * p.ah + j);
                            av[u] = *reinterpret_cast<const float2*>(p.actions + t * 2);
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int gi = gi0 + u * 256;
                            if (gi >= groups) continue;
                            const int t = r0 + gi / (p.ah / 4), j = (gi % (p.ah / 4)) * 4;
                            float4 v;
                            v.x = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(av[u].x, w0[u].x), __fmul_rn(av[u].y, w1[u].x)), bb[u].x), ps[u].x);
                            v.y = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(av[u].x, w0[u].y), __fmul_rn(av[u].y, w1[u].y)), bb[u].y), ps[u].y);
                            v.z = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(av[u].x, w0[u].z), __fmul_rn(av[u].y, w1[u].z)), bb[u].z), ps[u].z);
                            v.w = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(av[u].x, w0[u].w), __fmul_rn(av[u].y, w1[u].w)), bb[u].w), ps[u].w);
                            *reinterpret_cast<uint2*>(p.x + (int64_t)t * p.ah + j) = pack_bf16x4(v);
                        }
                    }
                    publish(p, o, et);
                }
            } else if (op.kind == OP_HEAD) {
                // delta = LN_f(e).Wh + bh; a = a + s*delta (model.cpp:590-598)
                if (blockIdx.x < op.n_items) {
                    if (et == 0) wait_count(p.done + op.dep, op.dep_count);
                    epi_bar();
                }
                for (int it = blockIdx.x; it < op.n_items; it += gridDim.x) {
                    const int row = it * 8 + ew;
                    if (row < p.M) {
                        // lane = 4 consecutive features per 128-wide chunk; 16 chunks
                        // (2048 features) of loads in flight per pass
                        const float* xr = p.e + (int64_t)row * p.ah;
                        const int nch = p.ah / 128;
                        float s = 0.f;
                        for (int c0 = 0; c0 < nch; c0 += 16) {
                            float4 v[16];
#pragma unroll
                            for (int u = 0; u < 16; ++u)
                                v[u] = c0 + u < nch ? ldcg4(xr + (c0 + u) * 128 + lane * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                            for (int u = 0; u < 16; ++u) s += (v[u].x + v[u].y) + (v[u].z + v[u].w);
                        }
                        const float mean = warp_sum(s) / (float)p.ah;
                        float var = 0.f, d0 = 0.f, d1 = 0.f;
                        for (int c0 = 0; c0 < nch; c0 += 16) {
                            float4 v[16];
#pragma unroll
                            for (int u = 0; u < 16; ++u)
                                v[u] = c0 + u < nch ? ldcg4(xr + (c0 + u) * 128 + lane * 4) : make_float4(mean, mean, mean, mean);
#pragma unroll
                            for (int u = 0; u < 16; ++u) {
                                const float a0 = v[u].x - mean, a1 = v[u].y - mean, a2 = v[u].z - mean, a3 = v[u].w - mean;
                                var += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
                            }
                        }
                        const float inv = 1.0f / sqrtf(warp_sum(var) / (float)p.ah + 1e-5f);
                        for (int c0 = 0; c0 < nch; c0 += 16) {
                            float4 v[16];
                            float4 wa[16], wb2[16];
#pragma unroll
                            for (int u = 0; u < 16; ++u) {
                                const bool ok = c0 + u < nch;
                                const int j = (c0 + u) * 128 + lane * 4;
                                v[u] = ok ? ldcg4(xr + j) : make_float4(mean, mean, mean, mean);
                                wa[u] = ok ? *reinterpret_cast<const float4*>(p.w_head + j * 2) : make_float4(0.f, 0.f, 0.f, 0.f);
                                wb2[u] = ok ? *reinterpret_cast<const float4*>(p.w_head + j * 2 + 4) : make_float4(0.f, 0.f, 0.f, 0.f);
                            }
#pragma unroll
                            for (int u = 0; u < 16; ++u) {
                                const float y0 = (v[u].x - mean) * inv, y1 = (v[u].y - mean) * inv;
                                const float y2 = (v[u].z - mean) * inv, y3 = (v[u].w - mean) * inv;
                                d0 += y0 * wa[u].x + y1 * wa[u].z + y2 * wb2[u].x + y3 * wb2[u].z;
                                d1 += y0 * wa[u].y + y1 * wa[u].w + y2 * wb2[u].y + y3 * wb2[u].w;
                            }
                        }
                        d0 = warp_sum(d0);
                        d1 = warp_sum(d1);
                        if (lane == 0) {
                            const float delta0 = d0 + p.b_head[0], delta1 = d1 + p.b_head[1];
                            p.actions[row * 2] = __fadd_rn(p.actions[row * 2], __fmul_rn(p.update_scale, delta0));
                            p.actions[row * 2 + 1] =
                                __fadd_rn(p.actions[row * 2 + 1], __fmul_rn(p.update_scale, delta1));
                        }
                    }
                    publish(p, o, et);
                }
            } else if (op.kind == OP_GEMM) {
                const bool split_path = op.splits > 1;
                const bool ln_in = op.epi == EPI_LN_BF16 || op.epi == EPI_LN_GELU_BF16;
                const bool gelu = op.epi == EPI_GELU_BF16 || op.epi == EPI_LN_GELU_BF16;
                const bool resid = op.epi == EPI_RESID_F32;
                const bool f32o = resid || op.epi == EPI_F32;
                for (int it = blockIdx.x; it < op.n_items; it += gridDim.x) {
                    const int TNo = op.tn;
                    const GemmItem g = gemm_item(op, it, TNo);
                    // tokens this CTA finalises: the whole tile, or 1/S of it for a split
                    const int own_lo = split_path ? (g.s * TNo) / op.splits : 0;
                    const int own_hi = split_path ? ((g.s + 1) * TNo) / op.splits : TNo;
                    const int own_h = (own_hi - own_lo) / 2;  // per warp half
                    const int my_lo = own_lo + hh * own_h;    // this warp half's owned tokens
                    const int my_n = max(0, min(own_h, p.M - (g.t0 + my_lo)));
                    if ((!split_path && ln_in) || resid) {
                        // inputs of other CTAs (LN statistics, the residual rows)
                        if (et == 0) wait_count(p.done + op.dep, op.dep_count);
                        epi_bar();
                        if (ln_in && et < TNo) {
                            const int t = g.t0 + et;
                            float mu = 0.f, rs = 0.f;
                            if (t < p.M) ln_stats(p, op.stats_in, t, mu, rs);
                            mu_s[et] = mu;
                            rs_s[et] = rs;
                        }
                        if (resid) {
                            // stage the residual rows this thread finalises (its feature,
                            // its owned tokens) into TMEM columns 256 + token while the
                            // mainloop runs: the drain then never waits on L2
                            const int fe = g.f0 + q * 32 + lane;
                            const float* er = reinterpret_cast<const float*>(op.out) + (int64_t)(g.t0 + my_lo) * op.ldo + fe;
#pragma unroll 1
                            for (int c = 0; c < my_n; c += 16) {
                                uint32_t v0[8], v1[8];
                                const bool ok1 = c + 8 < my_n;
#pragma unroll
                                for (int j = 0; j < 8; ++j) {
                                    v0[j] = __float_as_uint(__ldcg(er + (int64_t)(c + j) * op.ldo));
                                    v1[j] = ok1 ? __float_as_uint(__ldcg(er + (int64_t)(c + 8 + j) * op.ldo)) : 0u;
                                }
                                tmem_st8(tbase + lane_off + 256 + my_lo + c, v0);
                                if (ok1) tmem_st8(tbase + lane_off + 256 + my_lo + c + 8, v1);
                            }
                            tmem_st_wait();
                        }
                        epi_bar();
                    }
                    const int f = g.f0 + q * 32 + lane;
                    const int fl = q * 32 + lane;  // feature within the tile
                    uint8_t* stg_base = smem + C::OFF_STG;
                    const float bf = split_path ? 0.f : op.bias[f];
                    const float cs = (ln_in && !split_path) ? op.colsum[f] : 0.f;
                    const int cb = hh * (TNo / 2);
                    const int64_t ldo = split_path ? op.nf : op.ldo;
                    mbar_wait(acc_full, nmma & 1);
                    if (et == 0) trace_ev(p, o, TR_ACC);
                    tc_fence_after();
                    {
                        DrainArgs da;
                        da.tacc = tbase + lane_off + cb;
                        da.testage = resid && !split_path ? tbase + lane_off + 256 + cb : 0xffffffffu;
                        da.ncol = min(TNo / 2, max(0, p.M - (g.t0 + cb)));
                        da.c0 = cb;
                        da.fl = fl;
                        da.q = q;
                        da.lane = lane;
                        da.gelu = gelu;
                        da.bf = bf;
                        da.cs = cs;
                        da.mu_s = ln_in ? mu_s : nullptr;
                        da.rs_s = rs_s;
                        da.ldo = ldo;
                        da.erow = f32o ? reinterpret_cast<float*>(op.out) + (int64_t)(g.t0 + cb) * ldo + f : nullptr;
                        da.stg = stg_base;
                        da.stg_panel = TNo * 128;
                        da.st_part = (f32o && op.stats_out) ? st_part : nullptr;
                        da.part = nullptr;
                        da.dbg = 0;
                        if (!split_path) {
                            drain(da, ln_in, gelu, resid, f32o, false);
                        } else {
                            // partials of the tokens other splits finalise: [cb, cb+TNo/2)
                            // minus [own_lo, own_hi), clipped to M
                            const int hi = min(cb + TNo / 2, p.M - g.t0);
                            const int r0a = cb, r0b = min(hi, own_lo);
                            const int r1a = max(cb, own_hi), r1b = hi;
                            float* part0 = p.ws + ((int64_t)g.s * p.M + g.t0) * ldo + f;
                            if (r0b > r0a) {
                                da.tacc = tbase + lane_off + r0a;
                                da.ncol = r0b - r0a;
                                da.part = part0 + (int64_t)r0a * ldo;
                                drain_t<false, false, false, false, false, true>(da);
                            }
                            if (r1b > r1a) {
                                da.tacc = tbase + lane_off + r1a;
                                da.ncol = r1b - r1a;
                                da.part = part0 + (int64_t)r1a * ldo;
                                drain_t<false, false, false, false, false, true>(da);
                            }
                        }
                    }
                    if (et == 0) trace_ev(p, o, TR_LOOP);
                    if (!split_path) {
                        // staged bf16 tile (output, or the residual's bf16 copy) -> TMA store
                        fence_proxy_async();
                        epi_bar();
                        if (et == 0) trace_ev(p, o, TR_BAR);
                        if (et == 0) {
                            const CUtensorMap* tmo = f32o ? op.tmXB : op.tmO;
                            tma_store_2d(tmo, stg_base, g.f0, g.t0);
                            tma_store_2d(tmo, stg_base + TNo * 128, g.f0 + 64, g.t0);
                            bulk_commit();
                        }
                    }
                    if (et == 0) trace_ev(p, o, TR_DRAIN);
                    tc_fence_before();
                    epi_bar();
                    if (et == 0) mbar_arrive(acc_empty);
                    ++nmma;
                    if (split_path) {
                        split_meet(p, op, o, p.splitc + op.split_base + g.tile, et);
                        // finalise the owned tokens in the TMEM layout: own partial from
                        // TMEM + the other splits' partials (fixed split order) + bias
                        // (+ staged residual) -> e, bf16 copy, row statistics
                        FixArgs fa;
                        fa.tacc = tbase + lane_off + my_lo;
                        fa.testage = tbase + lane_off + 256 + my_lo;
                        fa.ncol = my_n;
                        fa.c0 = my_lo;
                        fa.S = op.splits;
                        fa.s_own = g.s;
                        fa.ws = p.ws + (int64_t)(g.t0 + my_lo) * op.nf + f;
                        fa.split_stride = (int64_t)p.M * op.nf;
                        fa.nf = op.nf;
                        fa.bf = op.bias[f];
                        // outputs staged in smem, written by TMA tensor stores below
                        const int orows = own_hi - own_lo;
                        const bool staged = op.tmEs != nullptr;
                        fa.erow = reinterpret_cast<float*>(op.out) + (int64_t)(g.t0 + my_lo) * op.ldo + f;
                        fa.xrow = op.xb_out ? op.xb_out + (int64_t)(g.t0 + my_lo) * op.ldo + f : nullptr;
                        fa.ldo = op.ldo;
                        fa.e_stg = staged ? reinterpret_cast<float*>(smem + C::OFF_STG) : nullptr;
                        fa.x_stg = (staged && op.xb_out) ? smem + C::OFF_STG + orows * 512 : nullptr;
                        fa.rows = orows;
                        fa.r0 = my_lo - own_lo;
                        fa.st_part = op.stats_out ? st_part : nullptr;
                        fa.q = q;
                        fa.lane = lane;
                        if (resid) fix_t<true>(fa);
                        else fix_t<false>(fa);
                        fence_proxy_async();
                        epi_bar();
                        if (staged && et == 0 && g.t0 + own_lo < p.M) {
                            tma_store_2d(op.tmEs, smem + C::OFF_STG, g.f0, g.t0 + own_lo);
                            if (op.xb_out) {
                                tma_store_2d(op.tmXs, smem + C::OFF_STG + orows * 512, g.f0, g.t0 + own_lo);
                                tma_store_2d(op.tmXs, smem + C::OFF_STG + orows * 512 + orows * 128, g.f0 + 64,
                                             g.t0 + own_lo);
                            }
                            bulk_commit();
                        }
                        if (op.stats_out) {
                            epi_bar();
                            const int n_own = min(own_hi, p.M - g.t0) - own_lo;
                            if (et < n_own) {
                                const int c = own_lo + et;
                                float2 acc2 = st_part[c];
#pragma unroll
                                for (int qq = 1; qq < 4; ++qq) {
                                    const float2 v2 = st_part[qq * 256 + c];
                                    acc2.x += v2.x;
                                    acc2.y += v2.y;
                                }
                                op.stats_out[(int64_t)(g.t0 + c) * p.nft + g.f0 / 128] = acc2;
                            }
                        }
                    } else if (f32o && op.stats_out) {
                        // (sum, sumsq) of each row over this 128-feature tile: the 4
                        // lane quarters in a fixed order (deterministic)
                        if (et < TNo && g.t0 + et < p.M) {
                            float2 acc2 = st_part[et];
#pragma unroll
                            for (int qq = 1; qq < 4; ++qq) {
                                const float2 v2 = st_part[qq * 256 + et];
                                acc2.x += v2.x;
                                acc2.y += v2.y;
                            }
                            op.stats_out[(int64_t)(g.t0 + et) * p.nft + g.f0 / 128] = acc2;
                        }
                    }
                    publish(p, o, et);
                }
            } else if (op.kind == OP_ATTN) {
                const int i = q * 32 + lane;  // query row within the tile
                const float sl2 = p.alpha * 1.4426950408889634f;
                const uint32_t tS[2] = {tbase, tbase + 64};
                const uint32_t tOh = tbase + 128 + hh * HD;
                for (int it = blockIdx.x; it < op.n_items; it += gridDim.x) {
                    const AttnItem a = attn_item(op, it, p.M);
                    float m_ref = -INFINITY, l = 0.f;
                    for (int j = 0; j < a.nj; ++j) {
                        const uint32_t JJ = J + j, b = JJ & 1;
                        mbar_wait(&s_full[b], (JJ >> 1) & 1);
                        tc_fence_after();
                        uint32_t sr[32];
                        tmem_ld32(tS[b] + lane_off + hh * 32, sr);
                        tmem_ld_wait();
                        tc_fence_before();
                        mbar_arrive(&s_free[b]);
                        const int gb = a.g0 + j;
                        int lo = 0, hi = 32;
                        if (gb < op.nbp) {
                            hi = min(32, p.r - gb * 64 - hh * 32);
                        } else if ((i >> 6) != gb - op.nbp) {
                            hi = 0;  // another lane's action keys
                        }
                        float mx = -INFINITY;
#pragma unroll
                        for (int k = 0; k < 32; ++k) {
                            const float sv = (k >= lo && k < hi) ? __uint_as_float(sr[k]) * sl2 : -INFINITY;
                            sr[k] = __float_as_uint(sv);
                            mx = fmaxf(mx, sv);
                        }
                        // lazy rescale: the reference max only moves when the block
                        // max exceeds it by > 8 (log2 units); P <= 2^8 stays exact
                        float corr = 1.f;
                        if (m_ref == -INFINITY) {
                            m_ref = mx;
                        } else if (mx > m_ref + 8.f) {
                            corr = ex2(m_ref - mx);
                            m_ref = mx;
                        }
                        const float base = m_ref == -INFINITY ? 0.f : m_ref;
                        float rsum = 0.f;
                        uint32_t pk[16];
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            const float p0 = ex2(__uint_as_float(sr[2 * k]) - base);
                            const float p1 = ex2(__uint_as_float(sr[2 * k + 1]) - base);
                            rsum += p0 + p1;
                            __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
                            pk[k] = *reinterpret_cast<uint32_t*>(&b2);
                        }
                        l = l * corr + rsum;
                        if (JJ >= 2) mbar_wait(&p_free[b], ((JJ - 2) >> 1) & 1);
                        uint8_t* prow = smem + C::OFF_P + b * C::P_BYTES + i * 128;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const int ch = hh * 4 + c;
                            *reinterpret_cast<uint4*>(prow + ((ch ^ (i & 7)) << 4)) =
                                make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
                        }
                        fence_proxy_async();
                        if (__any_sync(0xffffffffu, corr != 1.f)) {
                            // O holds PV of blocks < j: wait for the last of them, rescale
                            mbar_wait(&p_free[(JJ - 1) & 1], ((JJ - 1) >> 1) & 1);
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
                        mbar_arrive(&p_full[b]);
                    }
                    J += a.nj;
                    // merge the two key halves of each row inside the CTA: exchange
                    // (m, l) through smem, then thread (row, half) combines dims
                    // [half*HD/2, (half+1)*HD/2) of O_A and O_B from TMEM
                    // (scratch overlaps the P tiles: only after the last PV completed)
                    mbar_wait(acc_full, nmma & 1);
                    if (et == 0) trace_ev(p, o, TR_ACC);
                    tc_fence_after();
                    float* mlx = reinterpret_cast<float*>(smem + C::OFF_SCR);  // [2][2][128]
                    mlx[(hh * 2 + 0) * 128 + i] = m_ref;
                    mlx[(hh * 2 + 1) * 128 + i] = l;
                    epi_bar();
                    const float m0 = mlx[i], l0 = mlx[128 + i], m1 = mlx[256 + i], l1 = mlx[384 + i];
                    const float mm = fmaxf(m0, m1);
                    const float w0 = m0 == -INFINITY ? 0.f : ex2(m0 - mm);
                    const float w1 = m1 == -INFINITY ? 0.f : ex2(m1 - mm);
                    const float lsum = w0 * l0 + w1 * l1;
                    const int t = a.row0 + i;
                    const bool final_out = op.splits == 1;
                    const float sc = final_out ? 1.0f / lsum : 1.0f;
                    constexpr int DH = HD / 2;  // dims per thread
#pragma unroll 1
                    for (int cc = 0; cc < DH; cc += 16) {
                        uint32_t oa[16], ob[16];
                        tmem_ld16(tbase + 128 + lane_off + hh * DH + cc, oa);
                        tmem_ld16(tbase + 128 + HD + lane_off + hh * DH + cc, ob);
                        tmem_ld_wait();
                        float v[16];
#pragma unroll
                        for (int e2 = 0; e2 < 16; ++e2)
                            v[e2] = (w0 * __uint_as_float(oa[e2]) + w1 * __uint_as_float(ob[e2])) * sc;
                        if (t < p.M) {
                            if (final_out) {
                                __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(op.out) + (int64_t)t * p.kv + a.h * HD + hh * DH + cc;
#pragma unroll
                                for (int e2 = 0; e2 < 16; e2 += 4)
                                    *reinterpret_cast<uint2*>(dst + e2) = pack_bf16x4(make_float4(v[e2], v[e2 + 1], v[e2 + 2], v[e2 + 3]));
                            } else {
                                float* dst = p.ws + ((int64_t)a.s * p.M + t) * p.kv + a.h * HD + hh * DH + cc;
#pragma unroll
                                for (int e2 = 0; e2 < 16; e2 += 4)
                                    *reinterpret_cast<float4*>(dst + e2) = make_float4(v[e2], v[e2 + 1], v[e2 + 2], v[e2 + 3]);
                            }
                        }
                    }
                    if (hh == 0 && t < p.M && !final_out) p.wsml[((int64_t)a.s * p.M + t) * p.H + a.h] = make_float2(mm, lsum);
                    tc_fence_before();
                    epi_bar();
                    if (et == 0) mbar_arrive(acc_empty);
                    ++nmma;
                    if (!final_out) {
                        split_meet(p, op, o, p.splitc + op.split_base + a.tile, et);
                        const int rb = a.row0 + (a.s * 128) / op.splits;
                        const int re = min(p.M, a.row0 + ((a.s + 1) * 128) / op.splits);
                        attn_fixup<HD>(p, op, a, rb, re, ew, lane);
                    }
                    publish(p, o, et);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tbase, 512);
}

}  // namespace mk
}  // namespace alpa
