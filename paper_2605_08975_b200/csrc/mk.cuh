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
// Warp roles (384 threads, 3 warpgroups): warp 0 TMA producer, warp 1 TMEM
// allocator + MMA issuer, warps 2-3 idle (warpgroup 0 gives its registers to
// the epilogue via setmaxnreg), warps 4..11 epilogue / softmax / elementwise
// (256 threads; TMEM lane quarter = warp & 3, column half = (warp - 4) >> 2).
#pragma once

#include "common.cuh"
#include "tc_gemm.cuh"

#include <type_traits>

namespace alpa {
namespace mk {

enum OpKind : int { OP_ENCODE = 0, OP_GEMM = 1, OP_ATTN = 2, OP_HEAD = 3 };
enum MkFlags : int { MK_NO_L2PF = 1, MK_NO_PRELOAD = 2, MK_L2_NORMAL = 8, MK_PRE_NORMAL = 16, MK_ATT_L2PF = 32 };

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
    const CUtensorMap* tmEs; // GEMM fp32 producer: split -> fp32 rows, box {128, TN/S}; unsplit -> SW128 box {32, TN, 1}
    const CUtensorMap* tmXs; // GEMM, split residual producer: bf16 copy, box {64, TN/S}
    const CUtensorMap* tmO16; // GEMM, unsplit: bf16 output (or the residual's bf16 copy), 16-row chunk x 2 panels
    const CUtensorMap* tmE16; // GEMM, unsplit fp32 output: 16-row chunk x 4 SW128 panels (chunk-major staging)
                             // attention: fp32 KV-split partials [S][M][kv], box {32, 128, 1} SW128
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
    // attention, multi topology (per-lane prefixes, pipeline.cpp:405-413): one
    // query tile per lane (rows 64..127 of the 128-row MMA tile are padding),
    // the lane's prefix K/V at rows ((lane_map[lane] * B + blk) * 2 [+1]) * r
    int multi, blk;
    int prows;               // attention: rows of the KV-split partial workspace per split
};

struct Params {
    const Op* ops;
    int n_ops;
    int* done;        // [n_ops] item completion counters (zeroed before each launch)
    int* splitc;      // per-tile split rendezvous counters
    float* ws;        // split partials (fp32)
    float2* wsml;     // attention (m, l) partials
    int M, ah, kv, H, r, nft;
    int B;                  // decoder blocks (prefix row arithmetic, multi topology)
    int rcap;               // prefix rows per K / V section (static capacity >= r)
    const int* lane_map;    // [N] prefix index per lane (multi topology)
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
    TR_FIXC0 = 16,   // split finalisation: chunk 0, 1, 2 of fix_t done (16..18)
    TR_FIXED = 19,   // split finalisation: fix_t returned
    TR_STORE = 20,   // split finalisation: staging fenced, TMA stores issued
    TR_STATS = 21,   // split finalisation: row statistics written
    TR_MERGE = 22,   // attention: key-half merge + partial stores done
    TR_FIXIN = 23,   // split finalisation: fix_t entered (slot 7 of FixArgs::tr)
    TR_FIXV0 = 24,   // split finalisation: chunk 0 values computed (slot 8)
    TR_SM0 = 25,     // attention: first S block ready (softmax starts)
    TR_SMX = 26,     // attention: softmax loop done
    TR_SMJ = 27,     // attention: softmax of block j done (27..31, j < 5)
    TR_SJ = 32,      // attention: S MMA of block j issued (32..36)
    TR_LJ = 37,      // attention: K/V block j loads issued (37..41)
    TR_FJ = 42,      // attention: K/V block j landed at the MMA issuer (42..46)
    TR_SX = 48,      // attention softmax of block 1 (thread 0): S ready, S read, exps, P slot free, P stored, arrived (48..53)
    // SM-clock (clock64) stamps (cycle-precise; the globaltimer ticks at 256 ns here).
    // Attention item pipeline, MMA thread and softmax thread et 0, block j < 6:
    TC_MSTART = 64,  // MMA: Q landed
    TC_MF = 65,      // MMA: K/V block j landed (65..70)
    TC_MS = 71,      // MMA: S_j issued (71..76)
    TC_MP = 77,      // MMA: P_j seen (77..82)
    TC_MPV = 83,     // MMA: PV_j issued (83..88)
    TC_SS = 89,      // softmax: S_j ready (89..94)
    TC_SR = 95,      // softmax: S_j in registers (95..100)
    TC_SE = 101,     // softmax: exps of block j done (101..106)
    TC_SPF = 107,    // softmax: P slot free (107..112)
    TC_SA = 113,     // softmax: P_j published (113..118)
    TC_ACC = 119,    // softmax: all MMAs of the item done
    TC_MERGE = 120,  // key-half merge + partial stores done
    // GEMM item, MMA thread: first stage landed, last MMA issued, cycles spent waiting
    // for landed stages after the first, k-blocks
    TC_G0 = 64, TC_G1 = 65, TC_GW = 66, TC_GK = 67,
    TR_NSLOT = 128,
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
    static constexpr int THREADS = 384;
    // setmaxnreg split of the launch allocation (384 x 168): warpgroup 0 (the
    // single-thread TMA / MMA roles) drops to 104, the 8 epilogue warps rise to
    // 200 (128 * 64 freed >= 256 * 32 taken; an inc the pool cannot cover blocks)
    static constexpr int REG_LO = 104;
    static constexpr int REG_HI = 200;
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

// Spin until *ctr >= want.  A schedule bug must not hang the GPU: after ~2^26
// polls (seconds) the kernel traps, the launch fails and the host reports it.
// Acquire polls without back-off: the observing load is the ordering load (a
// relaxed poll + sleep + final acquire cost one more L2 round trip per wait,
// measured -0.25 ms/scene).  The kernel keeps no data in L1, so the L1
// invalidation an acquire implies is free here.
__device__ inline int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
template <bool TR = false>
__device__ __forceinline__ void wait_count(const int* ctr, int want) {
    uint32_t n = 0;
    while (ld_acquire(ctr) < want) {
        if (++n > (1u << 26)) {
            // no call in the kernel's code (a call caps the setmaxnreg register budget):
            // the message naming the stalled counter is a debug build option
#ifdef ALPA_MK_WATCHDOG_PRINTF
            printf("alpa mk watchdog: block %d thread %d waits counter %p = %d < %d\n", blockIdx.x, threadIdx.x,
                   (const void*)ctr, ld_relaxed(ctr), want);
#endif
            __trap();
        }
    }
}

// Instrumentation (TR kernels only: the production kernel carries none of this
// code -- the kernel does not fit the instruction cache, every byte counts).
template <bool TR>
__device__ inline void stamp(const Params& p, int o) {
    if (TR && p.tstamp) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(p.tstamp + o, t);
    }
}

template <bool TR>
__device__ inline void trace_ev(const Params& p, int o, int ev) {
    if (TR && p.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[((size_t)o * gridDim.x + blockIdx.x) * TR_NSLOT + ev] = t;
    }
}

template <bool TR>
__device__ inline void trace_clk(const Params& p, int o, int ev) {
    if (TR && p.trace) p.trace[((size_t)o * gridDim.x + blockIdx.x) * TR_NSLOT + ev] = (unsigned long long)clock64();
}
template <bool TR>
__device__ inline void trace_val(const Params& p, int o, int ev, unsigned long long v) {
    if (TR && p.trace) p.trace[((size_t)o * gridDim.x + blockIdx.x) * TR_NSLOT + ev] = v;
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
    int rv;     // valid query rows of the 128-row tile
    int prow0;  // first row of the tile in the KV-split partial workspace
};
__device__ inline AttnItem attn_item(const Op& op, int it, int M) {
    AttnItem a;
    a.s = it % op.splits;
    a.tile = it / op.splits;
    a.h = a.tile % op.tiles_f;
    a.qt = a.tile / op.tiles_f;
    // shared prefix: a tile = two lanes (128 rows); multi topology: one lane
    a.row0 = op.multi ? a.qt * 64 : a.qt * 128;
    a.rv = op.multi ? 64 : (M - a.row0 < 128 ? M - a.row0 : 128);
    a.prow0 = op.multi ? a.qt * 128 : a.row0;
    const int lanes = a.rv / 64;
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
    rs = rsqrtf(var + 1e-5f);  // MUFU, no IEEE slow-path call in the kernel
}

__device__ inline uint2 pack_bf16x4(float4 v) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    return pk;
}

// Merge the S KV-split partials of rows [rb, re) of one (head, query tile):
// log-sum-exp weights, fixed split order.  Flat (row, 4-dim group) items, two
// per thread per pass, every partial load of a pass in flight at once.
template <int HD>
__device__ inline void attn_fixup(const Params& p, const Op& op, const AttnItem& a, int rb, int re, int et) {
    const int np = op.splits;
    constexpr int NQ = HD / 4;  // 4-dim groups per row
    const int items = (re - rb) * NQ;
#pragma unroll 1
    for (int base = 0; base < items; base += 3 * 256) {
        float2 ml[3][6];
        float4 v[3][6];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int idx = base + et + k * 256;
            const bool ok = idx < items;
            const int t = rb + idx / NQ, d = (idx % NQ) * 4;
            const int pr = a.prow0 + (t - a.row0);  // partial workspace row
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                const bool on = ok && q < np;
                ml[k][q] = on ? __ldcg(p.wsml + ((int64_t)q * op.prows + pr) * p.H + a.h) : make_float2(-INFINITY, 0.f);
                v[k][q] = on ? ldcg4(p.ws + ((int64_t)q * op.prows + pr) * p.kv + a.h * HD + d) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int idx = base + et + k * 256;
            if (idx >= items) continue;
            const int t = rb + idx / NQ, d = (idx % NQ) * 4;
            float mx = -INFINITY;
#pragma unroll
            for (int q = 0; q < 6; ++q) mx = fmaxf(mx, ml[k][q].x);
            float L = 0.f;
            float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                const float w = ml[k][q].x == -INFINITY ? 0.f : ex2(ml[k][q].x - mx);
                L += w * ml[k][q].y;
                o.x += w * v[k][q].x; o.y += w * v[k][q].y; o.z += w * v[k][q].z; o.w += w * v[k][q].w;
            }
            const float inv = __fdividef(1.0f, L);
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

// Drain of an unsplit GEMM accumulator (every bf16 / fp32 epilogue kind).
// TMEM is read in the 16x256b shape (the mma C-fragment layout): per 16-token
// chunk a thread holds 4 features (fa + 8k) x 4 tokens, so the bf16 tile goes
// to the SW128 staging with one stmatrix.trans per 8 tokens (16-byte rows, no
// per-element addressing) and the per-token row statistics need only a 3-round
// butterfly.  Straight-line per epilogue kind (uniform choices hoisted: a
// per-element branch serialises every element's dependency chain).
//   v = rs*(acc - mu*cs) + b   (mu = 0, rs = 1 without LayerNorm: exact)
//   v = e + v                  (staged residual in TMEM columns 256+)
//   GELU; fp32 store; bf16 staging; row statistics.
struct DrainArgs {
    uint32_t tacc, tres;     // TMEM of the warp's lane quarter at the half's first token (acc / residual)
    int ncol;                // tokens of this warp half, multiple of 16
    int nvalid;              // of which inside M
    int cb;                  // first token of the half (tile-local)
    int q, lane;
    float bf[4], cs[4];      // per feature fa + 8k
    const float* mu_s;       // LayerNorm (mu, rstd) per tile token
    const float* rs_s;
    float* eout;             // fp32 output at (tile token 0, feature fa) (row stride ldo) or null
    long long ldo;
    uint8_t* stg;            // bf16 staging (two SW128 panels of [TN][128 B]) or null
    uint8_t* estg;           // fp32 staging (four SW128 panels of [TN][32 fp32]) instead of eout, or null
    int tn;
    // progressive TMA stores: each 16-token chunk leaves as soon as the half's 4 warps staged it
    const CUtensorMap* tm16; // bf16 box {64, 16} or null (whole-tile store after the drain)
    const CUtensorMap* te16; // fp32 box {32, 16, 1} or null
    int f0, t0, hh;
    float2* st_part;         // row-stat partials [4][256] or null
    unsigned long long* clk; // diagnostics (traced twin, et 0): clock64 per chunk phase, or null
};
template <bool LN, bool GELU, bool RESID, bool F32, bool STATS>
__device__ __forceinline__ void drain_t(const DrainArgs& a) {
    const int tq = a.lane & 3, tr = a.lane >> 2;
    // stmatrix row addresses: matrix i = lane >> 3 (features 8i..), row j = lane & 7 (token)
    const int mj = a.lane & 7;
    const int chunk = (a.q & 1) * 4 + (a.lane >> 3);
    // staging layout: progressive stores (tm16) keep each 16-row chunk's panels together
    // ([chunk][panel][16 rows][128 B], one 3-D TMA store per chunk); whole-tile stores
    // use [panel][TN rows][128 B]
    const bool cm = a.tm16 != nullptr;
    const uint32_t sbase = a.stg ? smem_u32(a.stg) + (a.q >> 1) * (cm ? 2048 : a.tn * 128) : 0u;
#pragma unroll 1
    for (int c = 0; c < a.ncol; c += 16) {
        uint32_t A[8], B[8], RA[8], RB[8];
        tmem_ld16x256b_x2(a.tacc + c, A);
        tmem_ld16x256b_x2(a.tacc + (16u << 16) + c, B);
        if constexpr (RESID) {
            tmem_ld16x256b_x2(a.tres + c, RA);
            tmem_ld16x256b_x2(a.tres + (16u << 16) + c, RB);
        }
        tmem_ld_wait();
        if (a.clk && c < 64) a.clk[(c >> 4) * 4 + 0] = clock64();
        // v[k][m]: feature fa + 8k, token t_m = cb + c + (m >> 1) * 8 + 2 tq + (m & 1)
        float v[4][4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int ri = (m >> 1) * 4 + (m & 1);
            v[0][m] = __uint_as_float(A[ri]);
            v[1][m] = __uint_as_float(A[ri + 2]);
            v[2][m] = __uint_as_float(B[ri]);
            v[3][m] = __uint_as_float(B[ri + 2]);
        }
        float mu[4], rs[4];
        if constexpr (LN) {
            const int t0 = a.cb + c + 2 * tq;
            const float2 m0 = *reinterpret_cast<const float2*>(a.mu_s + t0);
            const float2 m1 = *reinterpret_cast<const float2*>(a.mu_s + t0 + 8);
            const float2 r0 = *reinterpret_cast<const float2*>(a.rs_s + t0);
            const float2 r1 = *reinterpret_cast<const float2*>(a.rs_s + t0 + 8);
            mu[0] = m0.x; mu[1] = m0.y; mu[2] = m1.x; mu[3] = m1.y;
            rs[0] = r0.x; rs[1] = r0.y; rs[2] = r1.x; rs[3] = r1.y;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                float x = LN ? rs[m] * (v[k][m] - mu[m] * a.cs[k]) + a.bf[k] : v[k][m] + a.bf[k];
                if constexpr (RESID) {
                    const int ri = (m >> 1) * 4 + (m & 1) + (k & 1) * 2;
                    x = __uint_as_float(k < 2 ? RA[ri] : RB[ri]) + x;
                }
                if constexpr (GELU) x = gelu_tanh(x);
                v[k][m] = x;
            }
        if constexpr (F32) {
            if (a.estg) {
                // fp32 tile -> SW128 staging (TMA-stored): the 8 rows x 2 chunks a warp
                // writes per register land on distinct banks; no scattered global stores
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int r = a.cb + c + (m >> 1) * 8 + 2 * tq + (m & 1);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int fq = a.q * 32 + tr + 8 * k;  // feature within the tile
                        const int off = cm ? (r >> 4) * 8192 + (fq >> 5) * 2048 + (r & 15) * 128
                                           : (fq >> 5) * (a.tn * 128) + r * 128;
                        *reinterpret_cast<float*>(a.estg + off + (((((fq & 31) >> 2) ^ (r & 7))) << 4) + (fq & 3) * 4) =
                            v[k][m];
                    }
                }
            } else {
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int tl = c + (m >> 1) * 8 + 2 * tq + (m & 1);  // token within the half
                if (tl < a.nvalid) {
                    float* d = a.eout + (long long)(a.cb + tl) * a.ldo + tr;
#pragma unroll
                    for (int k = 0; k < 4; ++k) stg(d + 8 * k, v[k][m]);
                }
            }
            }
        }
        if (a.stg) {
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                const int tok = a.cb + c + g * 8 + mj;
                stmatrix_x4_trans(sbase + (cm ? (tok >> 4) * 4096 + (tok & 15) * 128 : tok * 128) + ((chunk ^ (tok & 7)) << 4),
                                  pack_bf16x2(v[0][2 * g], v[0][2 * g + 1]), pack_bf16x2(v[1][2 * g], v[1][2 * g + 1]),
                                  pack_bf16x2(v[2][2 * g], v[2][2 * g + 1]), pack_bf16x2(v[3][2 * g], v[3][2 * g + 1]));
            }
        }
        if (a.clk && c < 64) a.clk[(c >> 4) * 4 + 1] = clock64();
        if (a.tm16) {
            // this chunk's 16 rows of the half are staged by its 4 warps: store them now
            // (the store overlaps the rest of the drain instead of trailing it)
            fence_proxy_async();
            asm volatile("bar.sync %0, 128;" ::"r"(3 + a.hh) : "memory");
            if (a.clk && c < 64) a.clk[(c >> 4) * 4 + 2] = clock64();
            if (a.q == 0 && a.lane == 0) {
                const int r = a.cb + c;
                tma_store_3d(a.tm16, a.stg + (r >> 4) * 4096, 0, a.t0 + r, a.f0 >> 6);
                if (a.te16) tma_store_3d(a.te16, a.estg + (r >> 4) * 8192, 0, a.t0 + r, a.f0 >> 5);
                bulk_commit();
            }
            if (a.clk && c < 64) a.clk[(c >> 4) * 4 + 3] = clock64();
        }
        if constexpr (STATS) {
            // per token: sum over the thread's 4 features, then over the 8 lanes
            // sharing tq (xor 4, 8, 16): fixed order, deterministic
            float s1[4], s2[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                s1[m] = (v[0][m] + v[1][m]) + (v[2][m] + v[3][m]);
                s2[m] = (v[0][m] * v[0][m] + v[1][m] * v[1][m]) + (v[2][m] * v[2][m] + v[3][m] * v[3][m]);
            }
#pragma unroll
            for (int off = 4; off < 32; off <<= 1)
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    s1[m] += __shfl_xor_sync(0xffffffffu, s1[m], off);
                    s2[m] += __shfl_xor_sync(0xffffffffu, s2[m], off);
                }
            if (tr == 0) {
#pragma unroll
                for (int m = 0; m < 4; ++m)
                    a.st_part[a.q * 256 + a.cb + c + (m >> 1) * 8 + 2 * tq + (m & 1)] = make_float2(s1[m], s2[m]);
            }
        }
    }
}

// Mode dispatch (each epilogue kind has its own straight-line instance).
__device__ inline void drain(const DrainArgs& a, bool ln, bool gelu, bool resid, bool f32, bool stats) {
    if (resid) drain_t<false, false, true, true, true>(a);
    else if (f32 && stats) drain_t<false, false, false, true, true>(a);
    else if (f32) drain_t<false, false, false, true, false>(a);
    else if (ln && gelu) drain_t<true, true, false, false, false>(a);
    else if (ln) drain_t<true, false, false, false, false>(a);
    else if (gelu) drain_t<false, true, false, false, false>(a);
    else drain_t<false, false, false, false, false>(a);
}

// Split-K finalisation of one thread's owned tokens (TMEM layout): own partial
// (TMEM) + the other splits' partials (L2 workspace, [tile][split][TN][128]
// fp32 blocks: constant 512 B row stride, so every load is base + immediate)
// in a FIXED order (own, then the others by split index: deterministic, graph
// == eager bitwise) + bias (+ staged residual) -> fp32 staging rows.
struct FixArgs {
    uint32_t tacc, testage;   // TMEM: own partial / staged residual at the first owned token
    int ncol;                 // owned tokens of this thread, multiple of 8
    const float* oth[3];      // other splits' partial rows at (first owned token, feature), null: none
    float bf;
    float* e_stg;             // fp32 staging at (first owned row of this thread, feature), row stride 128
    unsigned long long* tr;   // diagnostics: per-chunk completion times (et 0 only) or null
};
__device__ inline void tr_now(unsigned long long* p) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *p = t;
}
template <bool RESID, bool TR>
__device__ __forceinline__ void fix_t(const FixArgs& a) {
    if (TR && a.tr) tr_now(a.tr + 7);
    const float* o0 = a.oth[0];
    const float* o1 = a.oth[1];
    const float* o2 = a.oth[2];
    float* d = a.e_stg;
    // batches of 3 chunks (24 tokens: all a thread owns at TN 192, S 4): every
    // partial load of a batch is issued before the first is used -- one L2 round
    // trip per batch (needs the epilogue warps' 200-register budget)
#pragma unroll 1
    for (int c0 = 0; c0 < a.ncol; c0 += 24) {
        float pv[3][3][8];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const int c = c0 + ch * 8;
            const bool on = c < a.ncol;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                pv[ch][0][j] = (on && o0) ? __ldcg(o0 + (c + j) * 128) : 0.f;
                pv[ch][1][j] = (on && o1) ? __ldcg(o1 + (c + j) * 128) : 0.f;
                pv[ch][2][j] = (on && o2) ? __ldcg(o2 + (c + j) * 128) : 0.f;
            }
        }
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const int c = c0 + ch * 8;
            if (c >= a.ncol) break;
            uint32_t r[8], rv[8];
            tmem_ld8(a.tacc + c, r);
            if constexpr (RESID) tmem_ld8(a.testage + c, rv);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                float acc = __uint_as_float(r[j]);
                if (o0) acc += pv[ch][0][j];
                if (o1) acc += pv[ch][1][j];
                if (o2) acc += pv[ch][2][j];
                float x = acc + a.bf;
                if constexpr (RESID) x = __uint_as_float(rv[j]) + x;
                d[(c + j) * 128] = x;
            }
            if (TR && a.tr && c < 24) tr_now(a.tr + c / 8);
        }
    }
}

// Row pass over the fp32 staging rows of a split finalisation: (sum, sumsq)
// per row of the 128-feature tile (LayerNorm statistics of the consumer, fixed
// order) and the bf16 copy into the SW128 staging of a TMA store box {64, rows}.
// 4 threads per row; step m: thread p takes features [8(4m+p), 8(4m+p)+8), so a
// row's 4 threads read 128 contiguous bytes; odd rows read the two halves in
// the other order (the 8 threads of one LDS.128 phase hit 32 distinct banks).
__device__ inline void fix_rows(const float* e_stg, uint8_t* x_stg, int rows, int n_valid, float2* stats_row0,
                                int nft, int et) {
    const int row = et >> 2, part = et & 3;
    if (row >= rows) return;  // whole 4-thread groups: the shuffles stay converged
    const float* rp = e_stg + row * 128;
    const int h = (row & 1) * 4;
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const int c16 = m * 4 + part;  // 8-feature chunk of the tile
        const float4 a = *reinterpret_cast<const float4*>(rp + c16 * 8 + h);
        const float4 b = *reinterpret_cast<const float4*>(rp + c16 * 8 + (4 - h));
        const float4 u = h ? b : a, w = h ? a : b;
        s1 += ((u.x + u.y) + (u.z + u.w)) + ((w.x + w.y) + (w.z + w.w));
        s2 += ((u.x * u.x + u.y * u.y) + (u.z * u.z + u.w * u.w)) + ((w.x * w.x + w.y * w.y) + (w.z * w.z + w.w * w.w));
        if (x_stg) {
            const uint2 lo = pack_bf16x4(u), hi = pack_bf16x4(w);
            *reinterpret_cast<uint4*>(x_stg + (c16 >> 3) * (rows * 128) + row * 128 + (((c16 & 7) ^ (row & 7)) << 4)) =
                make_uint4(lo.x, lo.y, hi.x, hi.y);
        }
    }
    const unsigned grp = 0xfu << (threadIdx.x & 28);
    s1 += __shfl_xor_sync(grp, s1, 1);
    s2 += __shfl_xor_sync(grp, s2, 1);
    s1 += __shfl_xor_sync(grp, s1, 2);
    s2 += __shfl_xor_sync(grp, s2, 2);
    if (stats_row0 && part == 0 && row < n_valid) stats_row0[(int64_t)row * nft] = make_float2(s1, s2);
}

// Item outputs are complete: make them visible to later generic and TMA
// (async-proxy) readers, then count the item.
template <bool TR>
__device__ inline void publish(const Params& p, int o, int et) {
    if ((et & 127) == 0) {  // the TMA-store issuers (et 0, and et 128 for the drain's second half)
        if (et == 0) trace_ev<TR>(p, o, TR_FIX);
        bulk_wait_all();  // this item's TMA stores have landed
    }
    fence_proxy_async_global();
    epi_bar();
    if (et == 0) {
        trace_ev<TR>(p, o, TR_FENCE);
        red_release_add(p.done + o, 1);  // release is cumulative over the CTA's writes (bar.sync)
        trace_clk<TR>(p, o, 95);
        stamp<TR>(p, o);
        trace_ev<TR>(p, o, TR_PUB);
    }
}

// Split rendezvous: every split of a tile has written its partial.  Thread 0
// also acquires the op's input dependency, so the fixup may read rows other
// CTAs produced (residual stream, LayerNorm statistics).
template <bool TR>
__device__ inline void split_meet(const Params& p, const Op& op, int o, int* ctr, int et) {
    const int S = op.splits;
    epi_bar();
    if (et == 0) {
        if (op.dep >= 0) wait_count<TR>(p.done + op.dep, op.dep_count);
        red_release_add(ctr, 1);
        wait_count<TR>(ctr, S);
    }
    epi_bar();
    if (et == 0) trace_ev<TR>(p, o, TR_MEET);
}

// ------------------------------------------------------------------ the kernel
template <int TN, int HD, bool TR>
__global__ void __launch_bounds__(384, 1) iter_kernel(const __grid_constant__ Params p) {
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
        if (TR && p.tstamp) {
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
            mbar_init(&s_free[i], 8);  // one arrival per epilogue warp
            mbar_init(&p_full[i], 8);
            mbar_init(&p_free[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    // register reallocation at warpgroup granularity: the epilogue's fused
    // handlers keep every load of a pass in flight only above the 168-register
    // launch cap (a 384-thread CTA)
    if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::REG_LO));
    if (warp == 0) {
        // ================================================= TMA producer
        // the whole warp runs the producer loop (uniform control flow); one elected
        // lane issues each TMA load / expect_tx
        {
            uint32_t ks = 0, natt = 0;
            // weights and the prefix are streamed once per iteration: evict_first
            // keeps them from displacing the kernel's code and the activations in L2
            const uint64_t wpol = (p.flags & MK_L2_NORMAL) ? policy_evict_normal() : policy_evict_first();
            const uint64_t ppol = (p.flags & MK_PRE_NORMAL) ? policy_evict_normal() : wpol;  // prefix K/V
            auto slot_acquire = [&](uint32_t kk) -> uint8_t* {
                const uint32_t st = kk % C::STAGES, ph = (kk / C::STAGES) & 1;
                mbar_wait(&empty[st], ph ^ 1);
                return smem + st * C::SLOT;
            };
            for (int o = 0; o < p.n_ops; ++o) {
                const Op op = p.ops[o];  // register copy: stores must not force reloads
                if (op.kind == OP_GEMM) {
                    if (lane == 0) tma_prefetch(op.tmW);
                    if (lane == 0) tma_prefetch(op.tmX);
                    bool waited = false;
                    for (int it = blockIdx.x; it < op.n_items; it += gridDim.x) {
                        const GemmItem g = gemm_item(op, it, op.tn);
                        const uint32_t stage_tx = C::W_BYTES + op.tn * 128;
                        // weights do not depend on earlier ops: start them first
                        int pre = g.nkb < C::STAGES ? g.nkb : C::STAGES;
                        if (p.flags & MK_NO_PRELOAD) {
                            pre = 0;
                            if (!waited && op.dep >= 0) {
                                wait_count<TR>(p.done + op.dep, op.dep_count);
                                fence_proxy_async_global();
                                waited = true;
                            }
                        }
#pragma unroll 1
                        for (int i = 0; i < pre; ++i) {
                            const uint32_t st = (ks + i) % C::STAGES;
                            uint8_t* sb = slot_acquire(ks + i);
                            mbar_expect_tx_w(&full[st], stage_tx);
                            tma_load_2d_hint_w(sb, op.tmW, &full[st], (g.kb0 + i) * 64, g.f0, wpol);
                        }
                        if (lane == 0) trace_ev<TR>(p, o, TR_PRE);
                        if (!waited && op.dep >= 0) {
                            wait_count<TR>(p.done + op.dep, op.dep_count);
                            fence_proxy_async_global();
                            waited = true;
                        }
                        if (lane == 0) trace_ev<TR>(p, o, TR_DEP);
#pragma unroll 1
                        for (int i = 0; i < g.nkb; ++i) {
                            const uint32_t st = (ks + i) % C::STAGES;
                            uint8_t* sb = smem + st * C::SLOT;
                            if (i >= pre) {
                                sb = slot_acquire(ks + i);
                                mbar_expect_tx_w(&full[st], stage_tx);
                                tma_load_2d_hint_w(sb, op.tmW, &full[st], (g.kb0 + i) * 64, g.f0, wpol);
                            }
                            tma_load_2d_w(sb + C::W_BYTES, op.tmX, &full[st], (g.kb0 + i) * 64, g.t0);
                        }
                        ks += g.nkb;
                    }
                } else if (op.kind == OP_ATTN) {
                    if (lane == 0) tma_prefetch(op.tmW);
                    if (lane == 0) tma_prefetch(op.tmX);
                    if (lane == 0) tma_prefetch(op.tmQ);
                    bool waited = false;
                    for (int it = blockIdx.x; it < op.n_items; it += gridDim.x) {
                        const AttnItem a = attn_item(op, it, p.M);
                        // this tile's prefix K / V rows (multi topology: the lane's own prefix)
                        long long pre_k = op.pre_k_row, pre_v = op.pre_v_row;
                        if (op.multi) {
                            pre_k = ((long long)p.lane_map[a.qt] * p.B + op.blk) * 2 * p.rcap;
                            pre_v = pre_k + p.rcap;
                        }
                        auto load_block = [&](int j) {
                            const uint32_t st = (ks + j) % C::STAGES;
                            uint8_t* kb = slot_acquire(ks + j);
                            if (j < 5) if (lane == 0) trace_ev<TR>(p, o, TR_LJ + j);
                            uint8_t* vb = kb + C::KVB;
                            mbar_expect_tx_w(&full[st], 2 * C::KVB);
                            const int gb = a.g0 + j;
                            for (int pn = 0; pn < HD / 64; ++pn) {
                                const int col = a.h * HD + pn * 64;
                                if (gb < op.nbp) {
                                    tma_load_2d_hint_w(kb + pn * C::KPANEL, op.tmW, &full[st], col,
                                                     (int)(pre_k + gb * 64), ppol);
                                    tma_load_2d_hint_w(vb + pn * C::KPANEL, op.tmW, &full[st], col,
                                                     (int)(pre_v + gb * 64), ppol);
                                } else {
                                    const int row = a.row0 + (gb - op.nbp) * 64;
                                    tma_load_2d_w(kb + pn * C::KPANEL, op.tmX, &full[st], p.kv + col, row);
                                    tma_load_2d_w(vb + pn * C::KPANEL, op.tmX, &full[st], 2 * p.kv + col, row);
                                }
                            }
                        };
                        int pre = 0;
#pragma unroll 1
                        while (pre < a.nj && pre < C::STAGES && a.g0 + pre < op.nbp) load_block(pre++);
                        if (p.flags & MK_ATT_L2PF) {
                            // the item's remaining prefix blocks (beyond the ring) into L2 now,
                            // while the ring waits for the QKV dependency
#pragma unroll 1
                            for (int j = pre; j < a.nj && a.g0 + j < op.nbp; ++j)
#pragma unroll 1
                                for (int pn = 0; pn < HD / 64; ++pn) {
                                    if (lane == 0) tma_prefetch_box_2d(op.tmW, a.h * HD + pn * 64, (int)(pre_k + (a.g0 + j) * 64));
                                    if (lane == 0) tma_prefetch_box_2d(op.tmW, a.h * HD + pn * 64, (int)(pre_v + (a.g0 + j) * 64));
                                }
                        }
                        if (lane == 0) trace_ev<TR>(p, o, TR_PRE);
                        if (!waited && op.dep >= 0) {
                            wait_count<TR>(p.done + op.dep, op.dep_count);
                            fence_proxy_async_global();
                            waited = true;
                        }
                        if (lane == 0) trace_ev<TR>(p, o, TR_DEP);
                        if (natt > 0) mbar_wait(q_empty, (natt - 1) & 1);
                        mbar_expect_tx_w(q_full, C::Q_BYTES);
                        for (int pn = 0; pn < HD / 64; ++pn)
                            tma_load_2d_w(smem + C::OFF_Q + pn * C::QPANEL, op.tmQ, q_full,
                                        a.h * HD + pn * 64, a.row0);
#pragma unroll 1
                        for (int j = pre; j < a.nj; ++j) load_block(j);
                        ks += a.nj;
                        ++natt;
                    }
                }
                // one copy of the prefetch loop for both op kinds (code size)
                if ((op.kind == OP_GEMM || op.kind == OP_ATTN) && lane == 0 && !(p.flags & MK_NO_L2PF))
                    l2_share(op.pf_ptr, op.pf_bytes, wpol);
            }
        }
    } else if (warp == 1) {
        // ================================================= MMA issuer
        // the whole warp runs the issue loop (uniform control flow); one elected
        // lane issues each tcgen05.mma / commit
        {
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
                        unsigned long long wsum = 0;
#pragma unroll 1
                        for (int i = 0; i < g.nkb; ++i) {
                            const uint32_t st = (ks + i) % C::STAGES, ph = ((ks + i) / C::STAGES) & 1;
                            const long long w0 = TR ? clock64() : 0;
                            mbar_wait(&full[st], ph);
                            if (TR && i > 0) wsum += (unsigned long long)(clock64() - w0);
                            if (i == 0) if (lane == 0) trace_clk<TR>(p, o, TC_G0);
                            if (i == 0) if (lane == 0) trace_ev<TR>(p, o, TR_MMA0);
                            tc_fence_after();
                            uint8_t* sb = smem + st * C::SLOT;
                            const uint64_t da = sdesc_k_sw128(sb);
                            const uint64_t db = sdesc_k_sw128(sb + C::W_BYTES);
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                tc_mma_bf16_w(tbase, da + 2 * k, db + 2 * k, idesc, (i | k) != 0 ? 1u : 0u);
                            tc_commit_w(&empty[st]);
                        }
                        tc_commit_w(acc_full);
                        if (lane == 0) trace_clk<TR>(p, o, TC_G1);
                        if (lane == 0) trace_val<TR>(p, o, TC_GW, wsum);
                        if (lane == 0) trace_val<TR>(p, o, TC_GK, (unsigned long long)g.nkb);
                        if (lane == 0) trace_ev<TR>(p, o, TR_MMA1);
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
                        if (lane == 0) trace_clk<TR>(p, o, TC_MSTART);
                        tc_fence_after();
                        auto issue_pv = [&](uint32_t JJ, uint32_t st, bool first) {
                            mbar_wait(&p_full[JJ & 1], (JJ >> 1) & 1);
                            if (JJ - J < 6) if (lane == 0) trace_clk<TR>(p, o, TC_MP + (JJ - J));
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
                                    tc_mma_bf16_w(tO[hh], da, dbv, idO, (first && kk == 0) ? 0u : 1u);
                                }
                            tc_commit_w(&empty[st]);
                            tc_commit_w(&p_free[JJ & 1]);
                            if (JJ - J < 6) if (lane == 0) trace_clk<TR>(p, o, TC_MPV + (JJ - J));
                        };
                        uint32_t prev_st = 0;
#pragma unroll 1
                        for (int j = 0; j < a.nj; ++j) {
                            const uint32_t JJ = J + j;
                            const uint32_t st = (ks + j) % C::STAGES, ph = ((ks + j) / C::STAGES) & 1;
                            mbar_wait(&full[st], ph);
                            if (j == 0) if (lane == 0) trace_ev<TR>(p, o, TR_MMA0);
                            if (j < 5) if (lane == 0) trace_ev<TR>(p, o, TR_FJ + j);
                            if (j < 6) if (lane == 0) trace_clk<TR>(p, o, TC_MF + j);
                            if (JJ >= 2) mbar_wait(&s_free[JJ & 1], ((JJ - 2) >> 1) & 1);
                            tc_fence_after();
                            const uint8_t* kb = smem + st * C::SLOT;
#pragma unroll
                            for (int kk = 0; kk < HD / 16; ++kk) {
                                const uint64_t da = sdesc_k_sw128(smem + C::OFF_Q + (kk >> 2) * C::QPANEL) + 2 * (kk & 3);
                                const uint64_t db = sdesc_k_sw128(kb + (kk >> 2) * C::KPANEL) + 2 * (kk & 3);
                                tc_mma_bf16_w(tS[JJ & 1], da, db, idS, kk > 0 ? 1u : 0u);
                            }
                            tc_commit_w(&s_full[JJ & 1]);
                            if (j < 6) if (lane == 0) trace_clk<TR>(p, o, TC_MS + j);
                            if (j < 5) if (lane == 0) trace_ev<TR>(p, o, TR_SJ + j);
                            if (j == a.nj - 1) tc_commit_w(q_empty);
                            if (j > 0) issue_pv(JJ - 1, prev_st, j == 1);
                            prev_st = st;
                        }
                        if (a.nj > 0) issue_pv(J + a.nj - 1, prev_st, a.nj == 1);
                        else tc_commit_w(q_empty);
                        tc_commit_w(acc_full);
                        if (lane == 0) trace_ev<TR>(p, o, TR_MMA1);
                        ks += a.nj;
                        J += a.nj;
                        ++natt;
                        ++nmma;
                    }
                }
            }
        }
        __syncwarp();
    }
    // back to the launch count for the common exit path, only after the epilogue
    // warps have given theirs back (an early inc by the idle warps 2-3 would take
    // the registers the epilogue's inc waits for: deadlock)
    asm volatile("bar.sync 2, 384;" ::: "memory");
    asm volatile("setmaxnreg.inc.sync.aligned.u32 168;");
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::REG_HI));
        // ================================================= epilogue / softmax / elementwise
        const int et = threadIdx.x - 128;  // 0..255
        const int ew = warp - 4;           // 0..7
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
                    const int r0 = it * op.tn, r1 = min(p.M, r0 + op.tn);  // op.tn = rows per item
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
                    publish<TR>(p, o, et);
                }
            } else if (op.kind == OP_HEAD) {
                // delta = LN_f(e).Wh + bh; a = a + s*delta (model.cpp:590-598)
                if (blockIdx.x < op.n_items) {
                    if (et == 0) wait_count<TR>(p.done + op.dep, op.dep_count);
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
                        const float inv = rsqrtf(warp_sum(var) / (float)p.ah + 1e-5f);
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
                    publish<TR>(p, o, et);
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
                        if (et == 0) wait_count<TR>(p.done + op.dep, op.dep_count);
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
                    const int cb = hh * (TNo / 2);
                    // unsplit drain: per-feature constants of the fragment layout (features fa + 8k)
                    float bfk[4] = {0.f, 0.f, 0.f, 0.f}, csk[4] = {0.f, 0.f, 0.f, 0.f};
                    if (!split_path) {
                        const int fa = g.f0 + q * 32 + (lane >> 2);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            bfk[k] = op.bias[fa + 8 * k];
                            if (ln_in) csk[k] = op.colsum[fa + 8 * k];
                        }
                    }
                    mbar_wait(acc_full, nmma & 1);
                    if (et == 0) trace_ev<TR>(p, o, TR_ACC);
                    if (et == 0) trace_clk<TR>(p, o, 68);
                    tc_fence_after();
                    {
                        if (!split_path) {
                            DrainArgs da;
                            da.tacc = tbase + lane_off + cb;
                            da.tres = tbase + lane_off + 256 + cb;
                            da.nvalid = min(TNo / 2, max(0, p.M - (g.t0 + cb)));
                            da.ncol = min(TNo / 2, (da.nvalid + 15) & ~15);
                            da.cb = cb;
                            da.q = q;
                            da.lane = lane;
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                da.bf[k] = bfk[k];
                                da.cs[k] = csk[k];
                            }
                            da.mu_s = mu_s;
                            da.rs_s = rs_s;
                            da.eout = f32o ? reinterpret_cast<float*>(op.out) + (int64_t)g.t0 * op.ldo + g.f0 + q * 32 : nullptr;
                            da.ldo = op.ldo;
                            da.stg = stg_base;
                            // unsplit residual producer with a staged fp32 map: e rows after the bf16 tile
                            da.estg = (f32o && op.tmEs) ? stg_base + TNo * 256 : nullptr;
                            da.tn = TNo;
                            da.st_part = st_part;
                            da.clk = (TR && p.trace && et == 0)
                                         ? p.trace + ((size_t)o * gridDim.x + blockIdx.x) * TR_NSLOT + 72
                                         : nullptr;
                            da.tm16 = op.tmO16;
                            da.te16 = (f32o && op.tmEs) ? op.tmE16 : nullptr;
                            da.f0 = g.f0;
                            da.t0 = g.t0;
                            da.hh = hh;
                            drain(da, ln_in, gelu, resid, f32o, f32o && op.stats_out);
                        } else {
                            // partials of the tokens other splits finalise: [cb, cb+TNo/2)
                            // minus [own_lo, own_hi), clipped to M
                            const int hi = min(cb + TNo / 2, p.M - g.t0);
                            const int r0a = cb, r0b = min(hi, own_lo);
                            const int r1a = max(cb, own_hi), r1b = hi;
                            float* blk = p.ws + ((int64_t)(g.tile * op.splits + g.s) * TNo) * 128 + fl;
#pragma unroll 1
                            for (int seg = 0; seg < 2; ++seg) {
                                const int ra = seg ? r1a : r0a, rb = seg ? r1b : r0b;
#pragma unroll 1
                                for (int c = ra; c < rb; c += 8) {
                                    uint32_t r[8];
                                    tmem_ld8(tbase + lane_off + c, r);
                                    tmem_ld_wait();
#pragma unroll
                                    for (int j = 0; j < 8; ++j) stg(blk + (c + j) * 128, __uint_as_float(r[j]));
                                }
                            }
                        }
                    }
                    if (et == 0) trace_ev<TR>(p, o, TR_LOOP);
                    if (et == 0) trace_clk<TR>(p, o, 69);
                    if (!split_path && !op.tmO16) {
                        // staged bf16 tile (output, or the residual's bf16 copy) -> TMA store
                        fence_proxy_async();
                        epi_bar();
                        if (et == 0) trace_ev<TR>(p, o, TR_BAR);
                        if (et == 0) {
                            const CUtensorMap* tmo = f32o ? op.tmXB : op.tmO;
                            tma_store_2d(tmo, stg_base, g.f0, g.t0);
                            tma_store_2d(tmo, stg_base + TNo * 128, g.f0 + 64, g.t0);
                            if (f32o && op.tmEs) {
#pragma unroll 1
                                for (int pn = 0; pn < 4; ++pn)
                                    tma_store_3d(op.tmEs, stg_base + TNo * 256 + pn * (TNo * 128), g.f0 + 32 * pn, g.t0, 0);
                            }
                            bulk_commit();
                        }
                    }
                    if (et == 0) trace_ev<TR>(p, o, TR_DRAIN);
                    tc_fence_before();
                    epi_bar();
                    if (et == 0) mbar_arrive(acc_empty);
                    ++nmma;
                    if (split_path) {
                        if (et == 0) trace_clk<TR>(p, o, 90);
                        split_meet<TR>(p, op, o, p.splitc + op.split_base + g.tile, et);
                        if (et == 0) trace_clk<TR>(p, o, 91);
                        // finalise the owned tokens in the TMEM layout: own partial from
                        // TMEM + the other splits' partials + bias (+ staged residual) ->
                        // fp32 staging; then the row pass (stats + bf16 copy) and TMA stores
                        const int orows = own_hi - own_lo;
                        float* e_stg = reinterpret_cast<float*>(smem + C::OFF_STG);
                        uint8_t* x_stg = op.xb_out ? smem + C::OFF_STG + orows * 512 : nullptr;
                        FixArgs fa;
                        fa.tacc = tbase + lane_off + my_lo;
                        fa.testage = tbase + lane_off + 256 + my_lo;
                        fa.ncol = (my_n + 7) & ~7;
#pragma unroll
                        for (int k = 0; k < 3; ++k) {
                            const int sk = k < g.s ? k : k + 1;  // the other splits, by index
                            fa.oth[k] = sk < op.splits
                                            ? p.ws + ((int64_t)(g.tile * op.splits + sk) * TNo + my_lo) * 128 + fl
                                            : nullptr;
                        }
                        fa.bf = op.bias[f];
                        fa.e_stg = e_stg + (my_lo - own_lo) * 128 + fl;
                        fa.tr = (TR && p.trace && et == 0)
                                    ? p.trace + ((size_t)o * gridDim.x + blockIdx.x) * TR_NSLOT + TR_FIXC0
                                    : nullptr;
                        if (resid) fix_t<true, TR>(fa);
                        else fix_t<false, TR>(fa);
                        if (et == 0) trace_clk<TR>(p, o, 92);
                        if (et == 0) trace_ev<TR>(p, o, TR_FIXED);
                        // the fp32 rows leave while the row pass builds the stats and bf16 copy
                        fence_proxy_async();
                        epi_bar();
                        const int n_own = min(own_hi, p.M - g.t0) - own_lo;
                        if (et == 0 && n_own > 0) {
                            tma_store_2d(op.tmEs, smem + C::OFF_STG, g.f0, g.t0 + own_lo);
                            bulk_commit();
                        }
                        if (et == 0) trace_clk<TR>(p, o, 93);
                        fix_rows(e_stg, x_stg, orows, n_own,
                                 op.stats_out ? op.stats_out + (int64_t)(g.t0 + own_lo) * p.nft + g.f0 / 128 : nullptr,
                                 p.nft, et);
                        fence_proxy_async();
                        epi_bar();
                        if (et == 0 && n_own > 0 && x_stg) {
                            tma_store_2d(op.tmXs, x_stg, g.f0, g.t0 + own_lo);
                            tma_store_2d(op.tmXs, x_stg + orows * 128, g.f0 + 64, g.t0 + own_lo);
                            bulk_commit();
                        }
                        if (et == 0) trace_clk<TR>(p, o, 94);
                        if (et == 0) trace_ev<TR>(p, o, TR_STORE);
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
                    publish<TR>(p, o, et);
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
                        if (j == 0 && et == 0) trace_ev<TR>(p, o, TR_SM0);
                        if (j < 6 && et == 0) trace_clk<TR>(p, o, TC_SS + j);
                        const bool trj = TR && j == 1 && et == 0;
                        if (trj) trace_ev<TR>(p, o, TR_SX + 0);
                        tc_fence_after();
                        uint32_t sr[32];
                        tmem_ld32(tS[b] + lane_off + hh * 32, sr);
                        tmem_ld_wait();
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&s_free[b]);
                        if (trj) trace_ev<TR>(p, o, TR_SX + 1);
                        if (j < 6 && et == 0) trace_clk<TR>(p, o, TC_SR + j);
                        const int gb = a.g0 + j;
                        // keys of this (row, half) in the block: warp-uniform (a warp's 32 rows
                        // belong to one lane: i >> 6 = q >> 1); all 32 except the prefix tail
                        // block and the other lane's action block (none)
                        int hi = 32;
                        if (gb < op.nbp) hi = min(32, p.r - gb * 64 - hh * 32);
                        else if ((i >> 6) != gb - op.nbp) hi = 0;
                        if (i >= a.rv) hi = 0;  // padding rows (multi topology, ragged tail)
                        const float* srf = reinterpret_cast<const float*>(sr);
                        // block max of the raw scores (tree: no 32-deep dependency chain);
                        // max(s) * scale == max(s * scale) for scale > 0
                        float mx = -INFINITY;
                        if (hi == 32) {
                            float t8[8];
#pragma unroll
                            for (int k = 0; k < 8; ++k)
                                t8[k] = fmaxf(fmaxf(srf[4 * k], srf[4 * k + 1]), fmaxf(srf[4 * k + 2], srf[4 * k + 3]));
                            mx = fmaxf(fmaxf(fmaxf(t8[0], t8[1]), fmaxf(t8[2], t8[3])),
                                       fmaxf(fmaxf(t8[4], t8[5]), fmaxf(t8[6], t8[7]))) * sl2;
                        } else if (hi > 0) {
#pragma unroll
                            for (int k = 0; k < 32; ++k) {
                                if (k >= hi) sr[k] = __float_as_uint(-INFINITY);
                                mx = fmaxf(mx, __uint_as_float(sr[k]));
                            }
                            mx *= sl2;
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
                        const float nb = m_ref == -INFINITY ? 0.f : -m_ref;
                        float rsum = 0.f;
                        uint32_t pk[16];
                        if (hi > 0) {
                            float r4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                const float p0 = ex2(fmaf(srf[2 * k], sl2, nb));
                                const float p1 = ex2(fmaf(srf[2 * k + 1], sl2, nb));
                                r4[k & 3] += p0 + p1;
                                pk[k] = pack_bf16x2(p0, p1);
                            }
                            rsum = (r4[0] + r4[1]) + (r4[2] + r4[3]);
                        } else {
#pragma unroll
                            for (int k = 0; k < 16; ++k) pk[k] = 0u;
                        }
                        l = l * corr + rsum;
                        if (trj) trace_ev<TR>(p, o, TR_SX + 2);
                        if (j < 6 && et == 0) trace_clk<TR>(p, o, TC_SE + j);
                        if (JJ >= 2) mbar_wait(&p_free[b], ((JJ - 2) >> 1) & 1);
                        if (trj) trace_ev<TR>(p, o, TR_SX + 3);
                        if (j < 6 && et == 0) trace_clk<TR>(p, o, TC_SPF + j);
                        uint8_t* prow = smem + C::OFF_P + b * C::P_BYTES + i * 128;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const int ch = hh * 4 + c;
                            *reinterpret_cast<uint4*>(prow + ((ch ^ (i & 7)) << 4)) =
                                make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
                        }
                        fence_proxy_async();
                        if (trj) trace_ev<TR>(p, o, TR_SX + 4);
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
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&p_full[b]);
                        if (trj) trace_ev<TR>(p, o, TR_SX + 5);
                        if (j < 6 && et == 0) trace_clk<TR>(p, o, TC_SA + j);
                        if (et == 0 && j < 5) trace_ev<TR>(p, o, TR_SMJ + j);
                    }
                    J += a.nj;
                    if (et == 0) trace_ev<TR>(p, o, TR_SMX);
                    // merge the two key halves of each row inside the CTA: exchange
                    // (m, l) through smem, then thread (row, half) combines dims
                    // [half*HD/2, (half+1)*HD/2) of O_A and O_B from TMEM
                    // (scratch overlaps the P tiles: only after the last PV completed)
                    mbar_wait(acc_full, nmma & 1);
                    if (et == 0) trace_ev<TR>(p, o, TR_ACC);
                    if (et == 0) trace_clk<TR>(p, o, TC_ACC);
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
                    const float sc = final_out ? __fdividef(1.0f, lsum) : 1.0f;
                    constexpr int DH = HD / 2;  // dims per thread
                    // KV-split partials: staged as fp32 SW128 panels of 32 dims ([HD/32][128 rows][128 B],
                    // the Q/P region: every MMA of the item has completed) and written by TMA
                    // stores -- thread-per-row global stores would scatter 32 rows per instruction
                    uint8_t* pst = smem + C::OFF_Q;
                    if (!final_out) epi_bar();  // the (m, l) scratch is read before the staging overwrites it
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
                        if (final_out) {
                            if (i < a.rv) {
                                __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(op.out) + (int64_t)t * p.kv + a.h * HD + hh * DH + cc;
#pragma unroll
                                for (int e2 = 0; e2 < 16; e2 += 4)
                                    *reinterpret_cast<uint2*>(dst + e2) = pack_bf16x4(make_float4(v[e2], v[e2 + 1], v[e2 + 2], v[e2 + 3]));
                            }
                        } else {
                            const int d0 = hh * DH + cc;  // 16 dims = 4 chunks of one 32-dim panel
                            uint8_t* prow = pst + (d0 >> 5) * (128 * 128) + i * 128;
#pragma unroll
                            for (int e2 = 0; e2 < 16; e2 += 4) {
                                const int ch = ((d0 & 31) + e2) >> 2;
                                *reinterpret_cast<float4*>(prow + ((ch ^ (i & 7)) << 4)) =
                                    make_float4(v[e2], v[e2 + 1], v[e2 + 2], v[e2 + 3]);
                            }
                            if ((d0 & 31) == 16) {
                                // the half's 4 warps completed this 32-dim panel: store it now
                                fence_proxy_async();
                                asm volatile("bar.sync %0, 128;" ::"r"(3 + hh) : "memory");
                                if (q == 0 && lane == 0) {
                                    tma_store_3d(op.tmXs, pst + (d0 >> 5) * (128 * 128), a.h * HD + (d0 & ~31), a.prow0, a.s);
                                    bulk_commit();
                                }
                            }
                        }
                    }
                    if (hh == 0 && i < a.rv && !final_out)
                        p.wsml[((int64_t)a.s * op.prows + a.prow0 + i) * p.H + a.h] = make_float2(mm, lsum);
                    if (!final_out && (et & 127) == 0) {  // the two panel-store issuers
                        bulk_wait_all();
                        fence_proxy_async_global();
                    }
                    if (et == 0) trace_ev<TR>(p, o, TR_MERGE);
                    if (et == 0) trace_clk<TR>(p, o, TC_MERGE);
                    tc_fence_before();
                    epi_bar();
                    if (et == 0) mbar_arrive(acc_empty);
                    ++nmma;
                    if (!final_out) {
                        split_meet<TR>(p, op, o, p.splitc + op.split_base + a.tile, et);
                        const int R = op.multi ? 64 : 128;
                        const int rb = a.row0 + (a.s * R) / op.splits;
                        const int re = min(a.row0 + a.rv, a.row0 + ((a.s + 1) * R) / op.splits);
                        attn_fixup<HD>(p, op, a, rb, re, et);
                    }
                    publish<TR>(p, o, et);
                }
            }
        }
        asm volatile("setmaxnreg.dec.sync.aligned.u32 168;");
        asm volatile("bar.sync 2, 384;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tbase, 512);
}

}  // namespace mk
}  // namespace alpa
