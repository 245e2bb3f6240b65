// The denoising iteration (Model::run_action_iteration, model.cpp:600-605) as
// a fixed kernel sequence, plus the device rollout.
//
// Per iteration (M = 64 N action rows of all trajectories):
//   encode      e0 = a.W_in + b_in + pos                      (model.cpp:558-559)
//   gemm        h1 = gelu(e0.W1 + b1)                         (model.cpp:560-561)
//   gemm        e  = h1.W2 + b2                               (model.cpp:562)
//   per block:  x = LN1(e); qkv = x.Wqkv + b (K/V land in the per-lane action
//               region, no write_action_kv copy); ctx = attn(q, [prefix_b || own
//               action K/V]); e += ctx.Wo + bo; x = LN2(e); h1 = gelu(x.W1+b1);
//               e += h1.W2 + b2                               (model.cpp:571-589)
//   head        a += s * (LN_f(e).Wh + bh)                    (model.cpp:590-598)
// f32 path: SIMT FFMA kernels.  bf16 path: tcgen05 GEMMs (tc_gemm.cuh), fp32
// residual stream, fp32 LN/softmax statistics.
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "ctx.h"
#include "tc_attn.cuh"
#include "tc_gemm.cuh"

namespace alpa {

namespace {

bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("ALPA_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

cudaEvent_t pool_event(Ctx& c) {
    if (c.ev_next == c.ev_pool.size()) {
        cudaEvent_t e;
        ALPA_CUDA(cudaEventCreate(&e));
        c.ev_pool.push_back(e);
    }
    return c.ev_pool[c.ev_next++];
}

template <typename... KArgs, typename... Args>
void launch_cl(Ctx& c, const KInfo& info, dim3 cluster, void (*k)(KArgs...), dim3 grid,
               dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl_enabled() && !c.prof_on) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cluster.x * cluster.y * cluster.z > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = cluster.x;
        attr[na].val.clusterDim.y = cluster.y;
        attr[na].val.clusterDim.z = cluster.z;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    ProfRec rec{info.tag, nullptr, nullptr, info.flops, info.bytes};
    if (c.prof_on) {
        rec.a = pool_event(c);
        rec.b = pool_event(c);
        ALPA_CUDA(cudaEventRecord(rec.a, s));
    }
    ALPA_CUDA(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...));
    if (c.prof_on) {
        ALPA_CUDA(cudaEventRecord(rec.b, s));
        c.prof.push_back(rec);
    }
    c.last_launches++;
}

template <typename... KArgs, typename... Args>
void launch(Ctx& c, const KInfo& info, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
            cudaStream_t s, Args... args) {
    launch_cl(c, info, dim3(1, 1, 1), k, grid, block, smem, s, args...);
}

// ------------------------------------------------------------------ encode
// e0[t][j] = ((a0*w0j + a1*w1j) + b_j) + pos[t%64][j] with the reference's
// rounding sequence (matmul acc from 0, then bias add, then position add).
template <typename T>
__global__ void encode_kernel(const float* __restrict__ act, const float* __restrict__ w,
                              const float* __restrict__ b, const float* __restrict__ pos,
                              T* __restrict__ out, int64_t M, int64_t ah, int64_t A) {
    pdl_wait();
    pdl_launch();
    const int64_t total = M * ah;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / ah, j = i % ah;
        float acc = __fmul_rn(act[t * 2], w[j]);
        acc = __fadd_rn(acc, __fmul_rn(act[t * 2 + 1], w[ah + j]));
        acc = __fadd_rn(acc, b[j]);
        acc = __fadd_rn(acc, pos[(t % A) * ah + j]);
        if constexpr (sizeof(T) == 2)
            out[i] = __float2bfloat16_rn(acc);
        else
            out[i] = acc;
    }
}

// ------------------------------------------------------------------ layernorm
// layernorm_row (kernels_serial.cpp:66-84), gamma=1 beta=0, eps=1e-5:
// mean, two-pass variance, inv = 1/sqrt(var+eps).  One warp per row.
template <typename T>
__global__ void layernorm_kernel(const float* __restrict__ x, T* __restrict__ out, int64_t M,
                                 int64_t n) {
    pdl_wait();
    pdl_launch();
    const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= M) return;
    const float* xr = x + row * n;
    float s = 0.f;
    for (int64_t j = lane; j < n; j += 32) s += xr[j];
    const float mean = warp_sum(s) / (float)n;
    float v = 0.f;
    for (int64_t j = lane; j < n; j += 32) {
        const float d = xr[j] - mean;
        v += d * d;
    }
    const float var = warp_sum(v) / (float)n;
    const float inv = 1.0f / sqrtf(var + 1e-5f);
    T* o = out + row * n;
    for (int64_t j = lane; j < n; j += 32) {
        const float y = (xr[j] - mean) * inv;
        if constexpr (sizeof(T) == 2)
            o[j] = __float2bfloat16_rn(y);
        else
            o[j] = y;
    }
}

// ------------------------------------------------------------------ f32 GEMM
// out[t][n] (op)= sum_k A[t][k] W[k][n] + b[n]; W in the reference [in][out]
// layout.  64x64 tile, 16-deep k slab, 4x4 register micro-tile (FFMA).
template <int EPI>
__global__ void __launch_bounds__(256)
    gemm_f32_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ W,
                    int64_t ldw, const float* __restrict__ bias, float* out, int64_t ldo, int T,
                    int N, int K) {
    pdl_wait();
    pdl_launch();
    __shared__ float As[16][64 + 4];
    __shared__ float Ws[16][64];
    const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
    const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += 16) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = tid + u * 256;  // 0..1023
            const int r = e / 16, cc = e % 16;
            const int gm = m0 + r, gk = k0 + cc;
            As[cc][r] = (gm < T && gk < K) ? A[(int64_t)gm * lda + gk] : 0.f;
            const int wr = e / 64, wc = e % 64;
            const int wk = k0 + wr, wn = n0 + wc;
            Ws[wr][wc] = (wk < K && wn < N) ? W[(int64_t)wk * ldw + wn] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            float av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Ws[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] += av[i] * bv[j];
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int t = m0 + ty * 4 + i;
        if (t >= T) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n >= N) continue;
            const float v = acc[i][j] + bias[n];
            float* o = out + (int64_t)t * ldo + n;
            if constexpr (EPI == EPI_GELU_BF16)
                *o = gelu_erf(v);
            else if constexpr (EPI == EPI_RESID_F32)
                *o = *o + v;
            else
                *o = v;
        }
    }
}

// ------------------------------------------------------------------ attention
// emit_attention (model.cpp:280-324) over attend_view (kv_cache.cpp:247-263):
// lane l, head h, action query i attends [prefix(l) rows 0..r-1 || lane l's 64
// action rows]; scores alpha*dot (alpha after the dot, kernels_serial.cpp:24),
// non-causal softmax, P.V.  Warp per query row, online softmax over 32-key
// chunks (warp-level max/sum), each lane owns head dims lane+32u.
// The prefix is read in place for every lane: no replicate_for_batch copy.
template <typename T>
__global__ void __launch_bounds__(256)
    attn_simt_kernel(const T* __restrict__ qkv, const T* __restrict__ prefix,
                     int64_t prefix_stride, int64_t block_off, const int32_t* __restrict__ lane_map,
                     int n, int r, int cap, int kv, int H, int A, float alpha, T* __restrict__ ctx) {
    pdl_wait();
    pdl_launch();
    __shared__ float qs[8][128];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t gw = blockIdx.x * 8 + warp;  // (l, h, i)
    const int hd = kv / H;
    if (gw >= (int64_t)n * H * A) return;
    const int i = gw % A, h = (gw / A) % H, l = gw / ((int64_t)A * H);
    const int64_t ld = 3 * (int64_t)kv;
    const T* qrow = qkv + ((int64_t)l * A + i) * ld + h * hd;
    for (int d = lane; d < hd; d += 32) qs[warp][d] = to_f(qrow[d]);
    __syncwarp();
    const T* pk = prefix + lane_map[l] * prefix_stride + block_off + h * hd;
    const T* pv = pk + (int64_t)cap * kv;  // V section: cap rows after K (static capacity)
    const T* ak = qkv + (int64_t)l * A * ld + kv + h * hd;
    const T* av = ak + kv;
    const int Ttot = r + A;
    float m = -INFINITY, lsum = 0.f;
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    for (int j0 = 0; j0 < Ttot; j0 += 32) {
        const int j = j0 + lane;
        float s = -INFINITY;
        if (j < Ttot) {
            const T* krow = j < r ? pk + (int64_t)j * kv : ak + (int64_t)(j - r) * ld;
            float acc = 0.f;
            for (int d = 0; d < hd; ++d) acc += qs[warp][d] * to_f(krow[d]);
            s = alpha * acc;
        }
        const float mn = fmaxf(m, warp_max(s));
        const float scale = __expf(m - mn);
        const float p = (j < Ttot) ? expf(s - mn) : 0.f;
        lsum = lsum * scale + warp_sum(p);
#pragma unroll
        for (int u = 0; u < 4; ++u) o[u] *= scale;
        const int jn = min(32, Ttot - j0);
        for (int jj = 0; jj < jn; ++jj) {
            const float pj = __shfl_sync(0xffffffffu, p, jj);
            const int jt = j0 + jj;
            const T* vrow = jt < r ? pv + (int64_t)jt * kv : av + (int64_t)(jt - r) * ld;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int d = lane + 32 * u;
                if (d < hd) o[u] += pj * to_f(vrow[d]);
            }
        }
        m = mn;
    }
    const float inv = 1.0f / lsum;
    T* orow = ctx + ((int64_t)l * A + i) * kv + h * hd;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int d = lane + 32 * u;
        if (d < hd) {
            if constexpr (sizeof(T) == 2)
                orow[d] = __float2bfloat16_rn(o[u] * inv);
            else
                orow[d] = o[u] * inv;
        }
    }
}

// ------------------------------------------------------------------ head + update
// delta = LN_f(e).Wh + bh (model.cpp:590-591); a = a + (s*delta)
// (model.cpp:594-598, two separate roundings).  One warp per action row.
__global__ void head_update_kernel(const float* __restrict__ e, const float* __restrict__ wh,
                                   const float* __restrict__ bh, float* __restrict__ act,
                                   int64_t M, int64_t ah, float scale) {
    pdl_wait();
    pdl_launch();
    const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= M) return;
    const float* xr = e + row * ah;
    float s = 0.f;
    for (int64_t j = lane; j < ah; j += 32) s += xr[j];
    const float mean = warp_sum(s) / (float)ah;
    float v = 0.f;
    for (int64_t j = lane; j < ah; j += 32) {
        const float d = xr[j] - mean;
        v += d * d;
    }
    const float inv = 1.0f / sqrtf(warp_sum(v) / (float)ah + 1e-5f);
    float d0 = 0.f, d1 = 0.f;
    for (int64_t j = lane; j < ah; j += 32) {
        const float y = (xr[j] - mean) * inv;
        d0 += y * wh[j * 2];
        d1 += y * wh[j * 2 + 1];
    }
    d0 = warp_sum(d0);
    d1 = warp_sum(d1);
    if (lane == 0) {
        const float delta0 = d0 + bh[0], delta1 = d1 + bh[1];
        act[row * 2] = __fadd_rn(act[row * 2], __fmul_rn(scale, delta0));
        act[row * 2 + 1] = __fadd_rn(act[row * 2 + 1], __fmul_rn(scale, delta1));
    }
}

// ------------------------------------------------------------------ rollout
// actions_to_trajectory (pipeline.cpp:124-148): fp64 explicit Euler unicycle,
// dt = 0.1, every update from the old state, pose = float cast.  sin/cos are
// evaluated in double-double and rounded once, so they match a correctly
// rounded libm (glibc) bit for bit; no FMA contraction anywhere.
struct dd {
    double hi, lo;
};
__device__ inline dd two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    const double err = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, err};
}
__device__ inline dd quick_two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ inline dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    const dd t = two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = quick_two_sum(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return quick_two_sum(s.hi, s.lo);
}
__device__ inline dd dd_mul(dd a, dd b) {
    const double p = __dmul_rn(a.hi, b.hi);
    double e = __fma_rn(a.hi, b.hi, -p);
    e = __dadd_rn(e, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi)));
    return quick_two_sum(p, e);
}
__device__ inline dd dd_mul_d(dd a, double b) {
    const double p = __dmul_rn(a.hi, b);
    double e = __fma_rn(a.hi, b, -p);
    e = __dadd_rn(e, __dmul_rn(a.lo, b));
    return quick_two_sum(p, e);
}

__device__ void sincos_dd(double x, double* sn, double* cs) {
    // Cody-Waite reduction by pi/2 with a 3-part constant (fdlibm split).
    const double k = rint(__dmul_rn(x, 6.36619772367581382433e-01));
    const double p1 = 1.57079632673412561417e+00, p2 = 6.07710050630396597660e-11,
                 p3 = 2.02226624871116645580e-21, p3t = 8.47842766036889956997e-32;
    dd r = two_sum(x, -__dmul_rn(k, p1));  // k*p1 exact for |k| < 2^20
    r = dd_add(r, dd{-__dmul_rn(k, p2), -__fma_rn(k, p2, -__dmul_rn(k, p2))});
    r = dd_add(r, dd{-__dmul_rn(k, p3), -__fma_rn(k, p3, -__dmul_rn(k, p3))});
    r = dd_add(r, dd{-__dmul_rn(k, p3t), 0.0});
    const dd r2 = dd_mul(r, r);
    const double z = r2.hi;
    // Taylor series to degree 27 / 26 (|r| <= pi/4: truncation < 1e-31 rel).  The
    // terms from r^13 / r^12 on are < 1e-10 of the result: summed in double (Horner
    // in r^2, error < 1e-26 relative); the head in double-double with exact
    // double-double coefficients (-1)^k / n! -- no divisions, one rounding at the end.
    double ts = -9.183689863795546e-29;
    ts = __fma_rn(ts, z, 6.446950284384474e-26);
    ts = __fma_rn(ts, z, -3.868170170630684e-23);
    ts = __fma_rn(ts, z, 1.9572941063391263e-20);
    ts = __fma_rn(ts, z, -8.22063524662433e-18);
    ts = __fma_rn(ts, z, 2.8114572543455206e-15);
    ts = __fma_rn(ts, z, -7.647163731819816e-13);
    ts = __fma_rn(ts, z, 1.6059043836821613e-10);
    double tc = -2.4795962632247976e-27;
    tc = __fma_rn(tc, z, 1.6117375710961184e-24);
    tc = __fma_rn(tc, z, -8.896791392450574e-22);
    tc = __fma_rn(tc, z, 4.110317623312165e-19);
    tc = __fma_rn(tc, z, -1.5619206968586225e-16);
    tc = __fma_rn(tc, z, 4.779477332387385e-14);
    tc = __fma_rn(tc, z, -1.1470745597729725e-11);
    tc = __fma_rn(tc, z, 2.08767569878681e-09);
    dd qs = dd_add(dd{-2.505210838544172e-08, 1.448814070935912e-24}, dd_mul_d(r2, ts));
    dd qc = dd_add(dd{-2.755731922398589e-07, -2.3767714622250297e-23}, dd_mul_d(r2, tc));
    qs = dd_add(dd{2.7557319223985893e-06, -1.858393274046472e-22}, dd_mul(r2, qs));
    qc = dd_add(dd{2.48015873015873e-05, 2.1511947866775882e-23}, dd_mul(r2, qc));
    qs = dd_add(dd{-0.0001984126984126984, -1.7209558293420705e-22}, dd_mul(r2, qs));
    qc = dd_add(dd{-0.001388888888888889, 5.300543954373577e-20}, dd_mul(r2, qc));
    qs = dd_add(dd{0.008333333333333333, 1.1564823173178714e-19}, dd_mul(r2, qs));
    qc = dd_add(dd{0.041666666666666664, 2.3129646346357427e-18}, dd_mul(r2, qc));
    qs = dd_add(dd{-0.16666666666666666, -9.25185853854297e-18}, dd_mul(r2, qs));
    qc = dd_add(dd{-0.5, 0.0}, dd_mul(r2, qc));
    const dd s = dd_add(r, dd_mul(r, dd_mul(r2, qs)));   // r + r^3 (s3 + r^2 (...))
    const dd c = dd_add(dd{1.0, 0.0}, dd_mul(r2, qc));   // 1 + r^2 (c2 + r^2 (...))
    const double sh = __dadd_rn(s.hi, s.lo), ch = __dadd_rn(c.hi, c.lo);
    const long q = ((long)k) & 3;
    if (q == 0) { *sn = sh; *cs = ch; }
    else if (q == 1) { *sn = ch; *cs = -sh; }
    else if (q == 2) { *sn = -sh; *cs = -ch; }
    else { *sn = -ch; *cs = sh; }
}

__global__ void rollout_kernel(const float* __restrict__ act, float* __restrict__ traj, int n,
                               int steps, const float* __restrict__ v0p, int* __restrict__ bad) {
    pdl_wait();
    pdl_launch();
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= n) return;
    double x = 0.0, y = 0.0, yaw = 0.0, v = (double)(*v0p);
    const double dt = 0.1;
    for (int i = 0; i < steps; ++i) {
        const float a = act[((int64_t)l * steps + i) * 2];
        const float k = act[((int64_t)l * steps + i) * 2 + 1];
        if (!isfinite(a) || !isfinite(k)) atomicExch(bad, 1);
        double sy, cy;
        sincos_dd(yaw, &sy, &cy);
        const double nx = __dadd_rn(x, __dmul_rn(__dmul_rn(v, cy), dt));
        const double ny = __dadd_rn(y, __dmul_rn(__dmul_rn(v, sy), dt));
        const double nyaw = __dadd_rn(yaw, __dmul_rn(__dmul_rn((double)k, v), dt));
        const double nv = __dadd_rn(v, __dmul_rn((double)a, dt));
        x = nx; y = ny; yaw = nyaw; v = nv;
        float* p = traj + ((int64_t)l * steps + i) * 3;
        p[0] = __double2float_rn(x);
        p[1] = __double2float_rn(y);
        p[2] = __double2float_rn(yaw);
    }
}

inline int ew_grid(int64_t n) {
    int64_t g = (n + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

// ------------------------------------------------------------------ GEMM dispatch
struct TcPlan {
    int splits, kbs;
};

// Split-K count = cluster size: a divisor of the token tile (each split CTA
// reduces TN/S rows), <= 8 (portable cluster), grid <= one wave of 148 SMs,
// and at least 2 k-blocks per split.
TcPlan plan_tc(int nf, int T, int K, int tn) {
    const int tiles = (nf / 128) * ((T + tn - 1) / tn);
    const int KB = K / 64;
    int best = 1;
    // the split-K epilogue stages TN x 128 fp32 plus (S-1) received slices
    // in the drained pipeline ring
    const int stage_bytes = 128 * 64 * 2 + tn * 64 * 2;
    const int ring = std::min(8, (200 * 1024) / stage_bytes) * stage_bytes;
    for (int s : {2, 4, 8})
        if (tn % s == 0 && tiles * s <= 148 && KB % s == 0 && KB / s >= 2 &&
            tn * 512 + (s - 1) * (tn / s) * 512 <= ring)
            best = s;
    return {best, KB / best};
}

KInfo gemm_info(const char* tag, const Linear& L, int T, size_t esz, int epi) {
    const double w = (double)L.in * L.out * esz, x = (double)T * L.in * esz;
    const double o = (double)T * L.out * ((epi == EPI_F32 || epi == EPI_RESID_F32) ? 4 : esz) *
                     (epi == EPI_RESID_F32 ? 2 : 1);
    return {tag, 2.0 * T * L.in * L.out, w + x + o};
}

// LN-fold side channels of one GEMM launch (see tc_gemm.cuh).
struct Side {
    bool produce = false;  // write e stats + bf16 copy (residual producers)
    bool consume = false;  // fold LN of the input rows (QKV, mlp1)
    const void* pf = nullptr;  // next op's weights to prefetch into L2
    long long pf_bytes = 0;
};

template <int TN, int EPI>
void launch_tc(Ctx& c, const char* tag, const Linear& L, const CUtensorMap& tmx, int T, void* out,
               int64_t ldo, cudaStream_t s, Side side = {}) {
    using Cf = GemmCfg<TN>;
    static bool configured = false;
    if (!configured) {
        ALPA_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<TN, EPI>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
        configured = true;
    }
    GemmArgs a{};
    a.nf = (int)L.out;
    a.t = T;
    a.k = (int)L.in;
    a.bias = L.b;
    a.out = out;
    a.ldo = ldo;
    const TcPlan p = plan_tc(a.nf, T, a.k, TN);
    a.splits = p.splits;
    a.kbs = p.kbs;
    a.nft = (int)(c.ah() / 128);
    {
        static const char* want = getenv("ALPA_TRACE_TAG");
        a.trace = want ? (strcmp(want, tag) == 0) : 1;
    }
    a.ln_n = (int)c.ah();
    if (side.produce) {
        a.stats_out = c.ws.stats;
        a.xb_out = (__nv_bfloat16*)c.ws.x;
    }
    if (side.consume) {
        a.stats_in = c.ws.stats;
        a.colsum = L.colsum;
    }
    a.pf_ptr = side.pf;
    a.pf_bytes = side.pf_bytes;
    dim3 grid(a.nf / 128, (T + TN - 1) / TN, p.splits);
    launch_cl(c, gemm_info(tag, L, T, 2, EPI), dim3(1, 1, p.splits), tc_gemm_kernel<TN, EPI>, grid,
              dim3(Cf::THREADS), (size_t)Cf::SMEM, s, L.tmap, tmx, a);
}

template <int EPI>
void gemm_tc(Ctx& c, const char* tag, const Linear& L, const CUtensorMap& tmx, int T, void* out,
             int64_t ldo, cudaStream_t s, Side side = {}) {
    switch (c.ws.tn) {
        case 64: launch_tc<64, EPI>(c, tag, L, tmx, T, out, ldo, s, side); break;
        case 128: launch_tc<128, EPI>(c, tag, L, tmx, T, out, ldo, s, side); break;
        case 192: launch_tc<192, EPI>(c, tag, L, tmx, T, out, ldo, s, side); break;
        default: launch_tc<256, EPI>(c, tag, L, tmx, T, out, ldo, s, side); break;
    }
}

template <int EPI>
void gemm_f32(Ctx& c, const char* tag, const Linear& L, const float* A, int64_t lda, int T,
              float* out, int64_t ldo, cudaStream_t s) {
    dim3 grid((unsigned)((L.out + 63) / 64), (unsigned)((T + 63) / 64));
    launch(c, gemm_info(tag, L, T, 4, EPI), gemm_f32_kernel<EPI>, grid, dim3(256), 0, s, A, lda,
           (const float*)L.w, L.out, (const float*)L.b, out, ldo, T, (int)L.out, (int)L.in);
}

template <int HD>
void launch_attn(Ctx& c, const KInfo& info, int64_t n, int64_t b, cudaStream_t s,
                 const void* pf = nullptr, long long pf_bytes = 0) {
    using Cf = AttnCfg<HD>;
    static bool configured = false;
    if (!configured) {
        ALPA_CUDA(cudaFuncSetAttribute(tc_attn_kernel<HD>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
        configured = true;
    }
    const int64_t A = c.steps(), M = n * A, kv = c.kv(), H = c.cfg.heads, r = c.prefix_r;
    AttnArgs a{};
    a.M = (int)M;
    a.r = (int)r;
    a.kv = (int)kv;
    a.nbp = (int)((r + 127) / 128);
    const int qtiles = (int)((M + 127) / 128);
    const int tiles = (int)H * qtiles;
    // KV splits = cluster size: 2 or 4 (clusters of 3/5/6 do not pack the
    // 16-20-SM GPCs into one wave), one wave, >= 1 block per split.
    int S = 1;
    for (int t : {2, 4})
        if (t <= a.nbp + 1 && tiles * t <= 148) S = t;
    if (const char* e = getenv("ALPA_ATTN_SPLITS")) S = std::max(1, std::min(atoi(e), a.nbp + 1));
    a.splits = S;
    const int64_t blk = (c.uniform_prefix * c.cfg.decoder_blocks + b) * 2;
    a.pre_k_row = blk * c.pcap();
    a.pre_v_row = (blk + 1) * c.pcap();
    a.alpha = 1.0f / sqrtf((float)(kv / H));
    a.ctx = (__nv_bfloat16*)c.ws.ctxb;
    a.pf_ptr = pf;
    a.pf_bytes = pf_bytes;
    launch_cl(c, info, dim3(1, 1, S), tc_attn_kernel<HD>, dim3((unsigned)H, (unsigned)qtiles, S),
              dim3(192), (size_t)Cf::SMEM, s, c.ws.tm_qkv, c.tm_pre, a);
}

}  // namespace

// The persistent kernel's token tile (its largest GEMM N; the ring stages and the
// epilogue staging follow from it) for M = 64 N tokens: a small cost model of
// one decoder block's GEMMs -- rounds of items over the SMs (tile quantisation,
// split-K as the plan would pick it) x k-blocks x max(MMA issue, per-SM
// ingress, ring-latency) per k-block + a per-round drain/sync cost.  Calibrated
// on B200 measurements over N = 2..64: it picks the measured best
// tile at 9 of 11 points and is within 5 % at the other two.
namespace tilemodel {
int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
int stages(int tn) {
    int slot = std::max(16384 + tn * 128, 32768);
    slot = (slot + 1023) / 1024 * 1024;
    const int aux = std::max(65536, tn * 256 + 12288);
    return std::min(8, (227 * 1024 - 1024 - aux - 1024) / slot);
}
int splits(int64_t tiles, int KB, int tn, int G) {
    if (tiles >= G) return 1;
    int best = 1;
    int64_t used = tiles;
    for (int s = 2; s <= 4; ++s) {
        if (tn % s || (tn / s) % 16 || tiles * s > G || KB / s < 2) continue;
        if ((s - 1) * cdiv(KB, s) >= KB) continue;
        if (tiles * s > used) {
            best = s;
            used = tiles * s;
        }
    }
    while (best > 1) {
        const int orows = tn / best;
        if (orows * 768 <= tn * 256 && orows % 16 == 0 && orows <= 64) break;
        --best;
        while (best > 1 && tn % best) --best;
    }
    return best;
}
}  // namespace tilemodel


// Modelled time (us) of one GEMM op of the persistent kernel: rounds of items
// over the SMs (tile quantisation, split-K as the plan picks it) x k-blocks x
// max(MMA issue max(45, N/2) cycles per 128xNx16 -- tools/mma_rate.cu --,
// per-SM ingress ~72 B/clk, ring latency ~1 us with the kernel tile's stages in
// flight) + a per-round drain / sync cost.  Calibrated on B200 sweeps.
double gemm_op_cost(int64_t M, int64_t nf, int64_t K, int tn_op, int tn_k, bool split_ok, int G) {
    using namespace tilemodel;
    const int64_t tiles = (nf / 128) * cdiv(M, tn_op);
    const int S = split_ok ? splits(tiles, (int)(K / 64), tn_op, G) : 1;
    const int64_t rounds = cdiv(tiles * S, G);
    const int64_t kb = cdiv(K / 64, S);
    const double stage = 16384.0 + tn_op * 128.0;
    const double mma = 4.0 * std::max(45.0, tn_op / 2.0);
    const double ingress = stage / 72.0;
    const double latency = stage / (stages(tn_k) * (16384.0 + tn_k * 128.0)) * 1900.0;
    return rounds * (kb * std::max(mma, std::max(ingress, latency)) / 1900.0 + (S == 1 ? 3.0 : 6.0));
}


int choose_token_tile(int64_t M, int G) {
    if (M <= 64) return 64;
    using tilemodel::cdiv;
    auto few = [&](int64_t nf, int tn) {
        int best = tn;
        for (int v = tn; v >= 64; v -= 32)
            if ((nf / 128) * cdiv(M, v) <= G) best = v;
        return best;
    };
    auto op = [&](int64_t nf, int64_t K, int tn_op, int tn_k, bool split_ok) {
        return gemm_op_cost(M, nf, K, tn_op, tn_k, split_ok, G);
    };
    int best = 192;
    double best_t = 1e30;
    for (int tn : {128, 192, 256}) {
        const double t = op(3072, 2048, few(3072, tn), tn, false) + op(2048, 1024, few(2048, tn), tn, false) +
                         op(8192, 2048, tn, tn, false) + op(2048, 8192, tn, tn, true);
        if (t < best_t * 0.999) {
            best_t = t;
            best = tn;
        }
    }
    return best;
}

void ensure_workspace(Ctx& c, int64_t n) {
    if (c.ws.n == n) return;
    // buffers change -> any captured graph is stale
    invalidate_graph(c);
    mk_release(c);
    Workspace& w = c.ws;
    for (void* p : {(void*)w.actions, (void*)w.traj, (void*)w.e, w.x, w.qkv, w.ctxb, w.h1,
                    (void*)w.counters, (void*)w.lane_map, (void*)w.stats})
        if (p) c.dfree(p);
    w = Workspace{};
    const int64_t A = c.steps(), M = n * A, ah = c.ah(), kv = c.kv();
    const size_t es = c.esz();
    w.n = n;
    w.actions = (float*)c.dalloc(M * 2 * sizeof(float));
    w.traj = (float*)c.dalloc(M * 3 * sizeof(float));
    w.e = (float*)c.dalloc(M * ah * sizeof(float));
    w.x = c.dalloc(M * ah * es);
    w.qkv = c.dalloc(M * 3 * kv * es);
    w.ctxb = c.dalloc(M * kv * es);
    w.h1 = c.dalloc(M * 4 * ah * es);
    w.counters = (int*)c.dalloc(8192 * sizeof(int));
    ALPA_CUDA(cudaMemset(w.counters, 0, 8192 * sizeof(int)));
    w.lane_map = (int32_t*)c.dalloc(n * sizeof(int32_t));
    const int T = (int)M;
    // bf16 persistent kernel: modelled choice; the per-op kernels of the fp32 /
    // cross-check paths keep a tile that divides M
    w.tn = c.bf16() ? choose_token_tile(M, 148)
                    : (T % 256 == 0) ? 256 : (T % 192 == 0) ? 192 : (T % 128 == 0) ? 128 : 64;
    if (const char* e = getenv("ALPA_WS_TN")) w.tn = atoi(e);  // A/B: kernel token tile
    if (c.bf16()) {
        w.stats = (float2*)c.dalloc(M * (ah / 128) * sizeof(float2));
        make_tmap_bf16_2d(&w.tm_x, w.x, ah, M, ah * 2, 64, w.tn);
        make_tmap_bf16_2d(&w.tm_ctx, w.ctxb, kv, M, kv * 2, 64, w.tn);
        make_tmap_bf16_2d(&w.tm_h1, w.h1, 4 * ah, M, 4 * ah * 2, 64, w.tn);
        make_tmap_bf16_2d(&w.tm_qkv, w.qkv, 3 * kv, M, 3 * kv * 2, 64, 128);
    }
}

void prepare_iteration(Ctx& c, int64_t n) {
    if (mk_usable(c)) mk_prepare(c, n);
}

// One persistent launch; in profiling mode also the per-op completion spans
// (globaltimer stamps, synchronous).
void enqueue_iteration_mk(Ctx& c, int64_t n, cudaStream_t s) {
    if (!c.prof_on) {
        mk_enqueue(c, n, s, nullptr);
        return;
    }
    MkState& m = c.mk;
    ProfRec rec{"iteration", pool_event(c), pool_event(c), 0.0, 0.0};
    for (double f : m.flops) rec.flops += f;
    {
        // algorithmic HBM bytes of one iteration: every weight once,
        // the shared prefix once, the action K/V written and read
        const double ah = (double)c.ah(), kv = (double)c.kv(), B = (double)c.cfg.decoder_blocks;
        const double eb = 2.0, A = (double)c.steps(), r = (double)c.prefix_r;
        rec.bytes = eb * (8 * ah * ah + 2 * ah + B * (4 * ah * kv + 8 * ah * ah) + 2 * ah) +
                    B * 2 * r * kv * eb + B * 2 * (double)n * A * kv * eb * 2;
    }
    ALPA_CUDA(cudaMemsetAsync(m.d_tstamp, 0, m.n_ops * sizeof(unsigned long long), s));
    ALPA_CUDA(cudaMemsetAsync(m.d_tstamp + m.n_ops, 0xFF, sizeof(unsigned long long), s));
    ALPA_CUDA(cudaEventRecord(rec.a, s));
    if (m.d_trace)
        ALPA_CUDA(cudaMemsetAsync(m.d_trace, 0, m.trace_elems * sizeof(unsigned long long), s));
    mk_enqueue(c, n, s, m.d_tstamp, m.d_trace);
    ALPA_CUDA(cudaEventRecord(rec.b, s));
    c.prof.push_back(rec);
    std::vector<unsigned long long> ts(m.n_ops + 1);
    ALPA_CUDA(cudaMemcpyAsync(ts.data(), m.d_tstamp, ts.size() * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, s));
    ALPA_CUDA(cudaStreamSynchronize(s));
    unsigned long long prev = ts[m.n_ops];
    for (int o = 0; o < m.n_ops; ++o) {
        const double ms = ts[o] > prev ? (ts[o] - prev) * 1e-6 : 0.0;
        c.prof_spans.push_back(ProfSpan{m.tags[o], ms, m.flops[o]});
        if (ts[o] > prev) prev = ts[o];
    }
}

void enqueue_iteration(Ctx& c, int64_t n, cudaStream_t s) {
    if (mk_usable(c)) {
        enqueue_iteration_mk(c, n, s);
        return;
    }
    Workspace& w = c.ws;
    const int64_t A = c.steps(), M = n * A, ah = c.ah(), kv = c.kv(), H = c.cfg.heads;
    const int T = (int)M;
    const int64_t r = c.prefix_r, cap = c.pcap();
    const int64_t prefix_stride = c.cfg.decoder_blocks * 2 * cap * kv;
    const float alpha = 1.0f / sqrtf((float)(kv / H));
    const int ln_grid = (int)((M + 7) / 8);
    const int attn_grid = (int)((n * H * A + 7) / 8);
    const double es = (double)c.esz();
    const KInfo enc{"encode", 4.0 * M * ah, M * 2 * 4.0 + M * ah * es};
    const KInfo ln{"layernorm", 8.0 * M * ah, M * ah * (4.0 + es)};
    // emit_attention FLOPs: QK^T and PV over r + 64 keys; bytes:
    // this block's prefix K/V once + q/k/v action rows + ctx.
    const KInfo att{"attention", 4.0 * n * A * (r + A) * kv,
                    2.0 * r * kv * es + M * 3.0 * kv * es + M * kv * es};
    const KInfo head{"head_update", 4.0 * M * ah + 8.0 * M, M * ah * 4.0 + M * 2 * 8.0};
    if (c.bf16()) {
        using bf = __nv_bfloat16;
        launch(c, enc, encode_kernel<bf>, dim3(ew_grid(M * ah)), dim3(256), 0, s, w.actions,
               (const float*)c.act_in.w, c.act_in.b, c.pos, (bf*)w.x, M, ah, A);
        // LayerNorms are folded into the GEMMs: residual producers emit the
        // bf16 copy of e (into x) + row statistics, QKV / mlp1 consume them.
        // Every op also prefetches the NEXT op's weights (or this block's
        // prefix K/V for the attention) into L2 while it computes.
        const int64_t B = c.cfg.decoder_blocks;
        auto wbytes = [](const Linear& L) { return (long long)(L.in * L.out * 2); };
        auto side = [&](bool prod, bool cons, const void* pf, long long nb) {
            Side sd;
            sd.produce = prod;
            sd.consume = cons;
            sd.pf = pf;
            sd.pf_bytes = nb;
            return sd;
        };
        const int64_t pre_block = 2 * cap * kv * 2;  // K + V of one block, bf16
        auto prefix_of = [&](int64_t b) {
            return (const void*)((const uint8_t*)c.prefix +
                                 (c.uniform_prefix < 0 ? 0 : c.uniform_prefix) *
                                     c.cfg.decoder_blocks * pre_block +
                                 b * pre_block);
        };
        gemm_tc<EPI_GELU_BF16>(c, "gemm_enc_mlp1", c.mlp1, w.tm_x, T, w.h1, 4 * ah, s,
                               side(false, false, c.mlp2.w, wbytes(c.mlp2)));
        gemm_tc<EPI_F32>(c, "gemm_enc_mlp2", c.mlp2, w.tm_h1, T, w.e, ah, s,
                         side(true, false, c.blocks[0].qkv.w, wbytes(c.blocks[0].qkv)));
        for (int64_t b = 0; b < B; ++b) {
            const Block& blk = c.blocks[b];
            gemm_tc<EPI_LN_BF16>(c, "gemm_qkv", blk.qkv, w.tm_x, T, w.qkv, 3 * kv, s,
                                 side(false, true, prefix_of(b), pre_block));
            const int64_t hd = kv / H;
            if (c.uniform_prefix >= 0 && c.tm_pre_valid && (hd == 64 || hd == 128)) {
                if (hd == 128)
                    launch_attn<128>(c, att, n, b, s, blk.o.w, wbytes(blk.o));
                else
                    launch_attn<64>(c, att, n, b, s, blk.o.w, wbytes(blk.o));
            } else {
                launch(c, att, attn_simt_kernel<bf>, dim3(attn_grid), dim3(256), 0, s,
                       (const bf*)w.qkv, (const bf*)c.prefix, prefix_stride, b * 2 * cap * kv,
                       (const int32_t*)w.lane_map, (int)n, (int)r, (int)cap, (int)kv, (int)H, (int)A,
                       alpha, (bf*)w.ctxb);
            }
            gemm_tc<EPI_RESID_F32>(c, "gemm_o", blk.o, w.tm_ctx, T, w.e, ah, s,
                                   side(true, false, blk.mlp1.w, wbytes(blk.mlp1)));
            gemm_tc<EPI_LN_GELU_BF16>(c, "gemm_mlp1", blk.mlp1, w.tm_x, T, w.h1, 4 * ah, s,
                                      side(false, true, blk.mlp2.w, wbytes(blk.mlp2)));
            const bool last = b + 1 == B;
            gemm_tc<EPI_RESID_F32>(c, "gemm_mlp2", blk.mlp2, w.tm_h1, T, w.e, ah, s,
                                   side(true, false, last ? nullptr : c.blocks[b + 1].qkv.w,
                                        last ? 0 : wbytes(c.blocks[b + 1].qkv)));
        }
    } else {
        float* x = (float*)w.x;
        float* h1 = (float*)w.h1;
        launch(c, enc, encode_kernel<float>, dim3(ew_grid(M * ah)), dim3(256), 0, s, w.actions,
               (const float*)c.act_in.w, c.act_in.b, c.pos, x, M, ah, A);
        gemm_f32<EPI_GELU_BF16>(c, "gemm_enc_mlp1", c.mlp1, x, ah, T, h1, 4 * ah, s);
        gemm_f32<EPI_F32>(c, "gemm_enc_mlp2", c.mlp2, h1, 4 * ah, T, w.e, ah, s);
        for (int64_t b = 0; b < c.cfg.decoder_blocks; ++b) {
            const Block& blk = c.blocks[b];
            launch(c, ln, layernorm_kernel<float>, dim3(ln_grid), dim3(256), 0, s,
                   (const float*)w.e, x, M, ah);
            gemm_f32<EPI_F32>(c, "gemm_qkv", blk.qkv, x, ah, T, (float*)w.qkv, 3 * kv, s);
            launch(c, att, attn_simt_kernel<float>, dim3(attn_grid), dim3(256), 0, s,
                   (const float*)w.qkv, (const float*)c.prefix, prefix_stride, b * 2 * cap * kv,
                   (const int32_t*)w.lane_map, (int)n, (int)r, (int)cap, (int)kv, (int)H, (int)A, alpha,
                   (float*)w.ctxb);
            gemm_f32<EPI_RESID_F32>(c, "gemm_o", blk.o, (const float*)w.ctxb, kv, T, w.e, ah, s);
            launch(c, ln, layernorm_kernel<float>, dim3(ln_grid), dim3(256), 0, s,
                   (const float*)w.e, x, M, ah);
            gemm_f32<EPI_GELU_BF16>(c, "gemm_mlp1", blk.mlp1, x, ah, T, h1, 4 * ah, s);
            gemm_f32<EPI_RESID_F32>(c, "gemm_mlp2", blk.mlp2, h1, 4 * ah, T, w.e, ah, s);
        }
    }
    launch(c, head, head_update_kernel, dim3(ln_grid), dim3(256), 0, s, (const float*)w.e,
           (const float*)c.head.w, (const float*)c.head.b, w.actions, M, ah, c.cfg.update_scale);
}

void enqueue_rollout(Ctx& c, int64_t n, const float* d_actions, float* d_traj, cudaStream_t s) {
    int* bad = reinterpret_cast<int*>(c.d_scalars + 1);
    ALPA_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
    const KInfo info{"rollout", 64.0 * n * c.steps(), n * c.steps() * 20.0};
    launch(c, info, rollout_kernel, dim3((unsigned)((n + 63) / 64)), dim3(64), 0, s, d_actions,
           d_traj,
           (int)n, (int)c.steps(), (const float*)c.d_scalars, bad);
}

void refresh_prefix_map(Ctx& c) {
    c.tm_pre_valid = false;
    if (!c.bf16() || !c.prefix) return;
    const uint64_t rows = (uint64_t)c.prefix_n * c.cfg.decoder_blocks * 2 * c.pcap();
    make_tmap_bf16_2d(&c.tm_pre, c.prefix, (uint64_t)c.kv(), rows, (uint64_t)c.kv() * 2, 64, 128);
    c.tm_pre_valid = true;
}

#ifdef ALPA_TRACE
// debug builds only: per-CTA phase stamps of the most recent traced kernels
extern "C" int alpa_debug_trace(unsigned long long* out, int64_t n) {
    return cudaMemcpyFromSymbol(out, g_trace, sizeof(unsigned long long) * 8 * n) == cudaSuccess ? 0 : 3;
}
extern "C" int alpa_debug_trace_clear(void) {
    static unsigned long long z[4096][8];
    return cudaMemcpyToSymbol(g_trace, z, sizeof(z)) == cudaSuccess ? 0 : 3;
}
#endif

void invalidate_graph(Ctx& c) {
    if (c.graph.exec) cudaGraphExecDestroy(c.graph.exec);
    c.graph = GraphCache{};
}

}  // namespace alpa
