// Reasoning-stage KV producer: the language model's prefill and
// decode steps on the device, appending every token's K/V IN PLACE into the
// static-capacity buffer the action stage attends -- [lanes][B][2][cap][kv] in
// the context dtype, the exact layout the persistent kernel's TMA maps read --
// so the sealed reasoning needs no host round trip and no copy.
//
// Reference: Model::prefill (model.cpp:408-464), Model::decode_step
// (model.cpp:484-507), Model::logits_head (model.cpp:509-513), the ctx
// assembly and decode loop of Engine::reasoning_pass (pipeline.cpp:279-390),
// KvCache::append_reasoning / seal_reasoning (kv_cache.cpp:120-190), static
// capacity T + max_new_tokens (pipeline.cpp:281-286).  The vision encoder and
// the tokenizer stay on the caller's side: prefill takes the vision rows and
// the prompt token ids, exactly the two inputs reasoning_pass combines.
//
// Arithmetic: f32 throughout (LN, linears with the bias added after the
// product, erf GELU, softmax attention with the causal mask), like the
// reference's serial kernels (kernels_serial.cpp); the LM's own attention reads
// an f32 copy of the cache, so a bf16 context only rounds the copy the action
// stage consumes.  The widths are small (hidden 64 at every SURVEY config), so
// these are plain SIMT kernels; the decode step is one small launch sequence
// per token, like the reference's substrate replay.
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "ctx.h"

namespace alpa {
namespace {

int64_t lin_n(int64_t in, int64_t out) { return in * out + out; }
int64_t blk_n(int64_t w, int64_t kv) {
    return 3 * lin_n(w, kv) + lin_n(kv, w) + lin_n(w, 4 * w) + lin_n(4 * w, w);
}

// x[x_off + t*ldx][:] = source row t + pos[p0 + t*pstep]: embedding rows
// (ids) or caller rows, plus the sinusoid (pipeline.cpp:297-324, 371-386)
__global__ void rs_embed_rows(const float* __restrict__ table, const int32_t* __restrict__ ids,
                              const float* __restrict__ rows_in, const float* __restrict__ pos,
                              int64_t n, int h, int64_t p0, int64_t pstep, int64_t ldx, int64_t x_off,
                              float* __restrict__ x, const int64_t* __restrict__ dpos) {
    if (dpos) p0 += *dpos;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * h;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = e / h;
        const int j = (int)(e % h);
        const float v = ids ? table[(int64_t)ids[t] * h + j] : rows_in[t * h + j];
        x[x_off + t * ldx + j] = v + pos[(p0 + t * pstep) * h + j];
    }
}

// LayerNorm, gamma 1 / beta 0 (make_norm, model.cpp:83-88), two-pass variance
// (kernels_serial.cpp:66-84); warp per row.
__global__ void rs_layernorm(const float* __restrict__ x, float* __restrict__ out, int64_t rows, int n) {
    const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const float* xr = x + row * n;
    float s = 0.f;
    for (int j = lane; j < n; j += 32) s += xr[j];
    const float mean = warp_sum(s) / (float)n;
    float v = 0.f;
    for (int j = lane; j < n; j += 32) {
        const float d = xr[j] - mean;
        v += d * d;
    }
    const float inv = 1.0f / sqrtf(warp_sum(v) / (float)n + 1e-5f);
    for (int j = lane; j < n; j += 32) out[row * n + j] = (xr[j] - mean) * inv;
}

// out[t][o] (=, GELU, +=) A[t][:] . W[:][o] + b[o]; reference [in][out] W;
// thread per output, ascending k (emit_linear: product, then the bias).
enum { RS_PLAIN = 0, RS_GELU = 1, RS_RESID = 2 };
template <int EPI>
__global__ void rs_linear(const float* __restrict__ A, int64_t rows, int in, const float* __restrict__ W,
                          const float* __restrict__ b, int out, float* __restrict__ O) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * out;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = e / out;
        const int o = (int)(e % out);
        const float* a = A + t * in;
        float acc = 0.f;
        for (int k = 0; k < in; ++k) acc = fmaf(a[k], W[(int64_t)k * out + o], acc);
        const float v = acc + b[o];
        if constexpr (EPI == RS_GELU) O[e] = gelu_erf(v);
        else if constexpr (EPI == RS_RESID) O[e] = O[e] + v;
        else O[e] = v;
    }
}

// KvCache::append_reasoning (kv_cache.cpp:120-179), static layout: rows
// [pos0, pos0 + n) of lane l, block b, written in place (f32 working copy +
// the context-dtype copy the action stage reads).
template <typename T>
__global__ void rs_append(const float* __restrict__ k, const float* __restrict__ v, int64_t n, int lanes,
                          int64_t pos0, int64_t B, int64_t b, int64_t cap, int kv, float* __restrict__ kv32,
                          T* __restrict__ kvo, const int64_t* __restrict__ dpos) {
    if (dpos) pos0 += *dpos;
    const int64_t total = (int64_t)lanes * n * kv;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int d = (int)(e % kv);
        const int64_t t = (e / kv) % n, l = e / ((int64_t)kv * n);
        const int64_t kr = (((l * B + b) * 2 + 0) * cap + pos0 + t) * kv + d;
        const int64_t vr = (((l * B + b) * 2 + 1) * cap + pos0 + t) * kv + d;
        const float kk = k[(l * n + t) * kv + d], vv = v[(l * n + t) * kv + d];
        if (kv32) {
            kv32[kr] = kk;
            kv32[vr] = vv;
        }
        if constexpr (sizeof(T) == 2) {
            kvo[kr] = __float2bfloat16_rn(kk);
            kvo[vr] = __float2bfloat16_rn(vv);
        } else {
            kvo[kr] = kk;
            kvo[vr] = vv;
        }
    }
}

// emit_attention over the reasoning view (model.cpp:280-324, spec_from_view
// causal for prefill, full for the single decode query): query i of lane l
// sits at position pos0 + i and attends keys [0, pos0 + i]; scores alpha *
// dot, softmax, P.V.  Warp per (lane, query, head), online softmax over 32-key
// chunks, lane owns head dims lane + 32u.
__global__ void rs_attention(const float* __restrict__ q, int64_t nq, int lanes, int64_t pos0,
                             const float* __restrict__ kv32, int64_t B, int64_t b, int64_t cap, int kv,
                             int H, float alpha, float* __restrict__ ctx, const int64_t* __restrict__ dpos) {
    if (dpos) pos0 += *dpos;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t gw = blockIdx.x * (int64_t)(blockDim.x / 32) + warp;
    if (gw >= (int64_t)lanes * nq * H) return;
    const int h = (int)(gw % H);
    const int64_t i = (gw / H) % nq, l = gw / ((int64_t)H * nq);
    const int hd = kv / H;
    const float* qr = q + (l * nq + i) * kv + h * hd;
    const float* kb = kv32 + ((l * B + b) * 2 + 0) * cap * kv + h * hd;
    const float* vb = kv32 + ((l * B + b) * 2 + 1) * cap * kv + h * hd;
    const int64_t nk = pos0 + i + 1;
    float m = -INFINITY, lsum = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
    for (int64_t j0 = 0; j0 < nk; j0 += 32) {
        const int64_t j = j0 + lane;
        float s = -INFINITY;
        if (j < nk) {
            const float* kr = kb + j * kv;
            float acc = 0.f;
            for (int d = 0; d < hd; ++d) acc = fmaf(qr[d], kr[d], acc);
            s = alpha * acc;
        }
        const float mn = fmaxf(m, warp_max(s));
        const float sc = expf(m - mn);
        const float pj = j < nk ? expf(s - mn) : 0.f;
        lsum = lsum * sc + warp_sum(pj);
#pragma unroll
        for (int u = 0; u < 4; ++u) o[u] *= sc;
        const int jn = (int)min((int64_t)32, nk - j0);
        for (int jj = 0; jj < jn; ++jj) {
            const float pw = __shfl_sync(0xffffffffu, pj, jj);
            const float* vr = vb + (j0 + jj) * kv;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int d = lane + 32 * u;
                if (d < hd) o[u] = fmaf(pw, vr[d], o[u]);
            }
        }
        m = mn;
    }
    const float inv = 1.0f / lsum;
    float* orow = ctx + (l * nq + i) * kv + h * hd;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int d = lane + 32 * u;
        if (d < hd) orow[d] = o[u] * inv;
    }
}

__global__ void rs_bump(int64_t* dpos, int64_t by) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *dpos += by;
}

// last row of every lane -> out (ReadSlice, model.cpp:454-463)
__global__ void rs_last_rows(const float* __restrict__ x, int64_t n, int lanes, int h, float* __restrict__ out) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < lanes * h; e += gridDim.x * blockDim.x) {
        const int l = e / h, j = e % h;
        out[e] = x[((int64_t)l * n + n - 1) * h + j];
    }
}

int grid_of(int64_t n) {
    const int64_t g = (n + 255) / 256;
    return (int)(g > 148 * 16 ? 148 * 16 : (g < 1 ? 1 : g));
}

void check_launch() { ALPA_CUDA(cudaGetLastError()); }

// The LM weights (token_embed, language blocks, lm_head) at their offsets in
// the one splitmix64 stream (ModelWeights::build, model.cpp:120-151).
void ensure_lm_weights(Ctx& c) {
    Reasoner& R = c.rs;
    if (R.weights) return;
    const alpa_model_cfg& m = c.cfg;
    const int64_t h = m.hidden_dim, kv = m.kv_dim, V = m.vocab_size, B = m.decoder_blocks;
    const int64_t patch_dim = m.patch_size * m.patch_size * 3;
    int64_t off = lin_n(patch_dim, h) + m.vision_blocks * blk_n(h, kv);
    auto f = [&](int64_t n) { return (float*)c.dalloc((size_t)n * sizeof(float)); };
    R.embed = f(V * h);
    draw_array_f32(c, off, V * h, R.embed);
    off += V * h;
    R.blocks.resize(B);
    for (int64_t b = 0; b < B; ++b) {
        LangBlock& L = R.blocks[b];
        auto lin = [&](float*& w, float*& bias, int64_t in, int64_t out) {
            w = f(in * out);
            bias = f(out);
            draw_linear_f32(c, off, in, out, w, bias);
            off += lin_n(in, out);
        };
        lin(L.wq, L.bq, h, kv);  // draw_block order: q, k, v, o, mlp1, mlp2 (model.cpp:90-101)
        lin(L.wk, L.bk, h, kv);
        lin(L.wv, L.bv, h, kv);
        lin(L.wo, L.bo, kv, h);
        lin(L.w1, L.b1, h, 4 * h);
        lin(L.w2, L.b2, 4 * h, h);
    }
    R.lm_w = f(h * V);
    R.lm_b = f(V);
    draw_linear_f32(c, off, h, V, R.lm_w, R.lm_b);
    ALPA_CUDA(cudaStreamSynchronize(c.stream));
    R.weights = true;
}

void ensure_rows(Ctx& c, int64_t rows) {
    Reasoner& R = c.rs;
    if (rows <= R.rows_cap) return;
    const int64_t h = c.cfg.hidden_dim, kv = c.cfg.kv_dim;
    for (float* p : {R.x, R.xn, R.q, R.k, R.v, R.att, R.h1})
        if (p) c.dfree(p);
    auto f = [&](int64_t n) { return (float*)c.dalloc((size_t)n * sizeof(float)); };
    R.x = f(rows * h);
    R.xn = f(rows * h);
    R.q = f(rows * kv);
    R.k = f(rows * kv);
    R.v = f(rows * kv);
    R.att = f(rows * kv);
    R.h1 = f(rows * 4 * h);
    R.rows_cap = rows;
}

void ensure_ids(Ctx& c, int64_t n) {
    Reasoner& R = c.rs;
    if (n <= R.ids_cap) return;
    if (R.ids) c.dfree(R.ids);
    R.ids = (int32_t*)c.dalloc((size_t)n * sizeof(int32_t));
    R.ids_cap = n;
}

// The language blocks over n new positions [pos0, pos0 + n) of every lane
// (rows = lanes * n in R.x), appending their K/V, then LN_f of each lane's
// last row and the logits head (model.cpp:429-464, 484-513).
// dpos: device position added to pos0 (decode: the graph-captured step reads the
// cache length from the device, so one captured step serves every token)
void lm_forward(Ctx& c, int64_t n, int64_t pos0, const int64_t* dpos) {
    Reasoner& R = c.rs;
    const alpa_model_cfg& m = c.cfg;
    const int64_t h = m.hidden_dim, kv = m.kv_dim, V = m.vocab_size, B = m.decoder_blocks, H = m.heads;
    const int64_t rows = R.lanes * n;
    const int L = (int)R.lanes;
    cudaStream_t s = c.stream;
    const float alpha = 1.0f / sqrtf((float)(kv / H));
    float* kv32 = c.bf16() ? R.kv32 : (float*)R.kv;
    const int ln_grid = (int)((rows + 7) / 8);
    for (int64_t b = 0; b < B; ++b) {
        const LangBlock& W = R.blocks[b];
        rs_layernorm<<<ln_grid, 256, 0, s>>>(R.x, R.xn, rows, (int)h);
        rs_linear<RS_PLAIN><<<grid_of(rows * kv), 256, 0, s>>>(R.xn, rows, (int)h, W.wq, W.bq, (int)kv, R.q);
        rs_linear<RS_PLAIN><<<grid_of(rows * kv), 256, 0, s>>>(R.xn, rows, (int)h, W.wk, W.bk, (int)kv, R.k);
        rs_linear<RS_PLAIN><<<grid_of(rows * kv), 256, 0, s>>>(R.xn, rows, (int)h, W.wv, W.bv, (int)kv, R.v);
        if (c.bf16())
            rs_append<__nv_bfloat16><<<grid_of(rows * kv), 256, 0, s>>>(
                R.k, R.v, n, L, pos0, B, b, R.cap, (int)kv, R.kv32, (__nv_bfloat16*)R.kv, dpos);
        else
            rs_append<float><<<grid_of(rows * kv), 256, 0, s>>>(R.k, R.v, n, L, pos0, B, b, R.cap, (int)kv,
                                                                nullptr, (float*)R.kv, dpos);
        rs_attention<<<(int)((rows * H + 7) / 8), 256, 0, s>>>(R.q, n, L, pos0, kv32, B, b, R.cap, (int)kv,
                                                               (int)H, alpha, R.att, dpos);
        rs_linear<RS_RESID><<<grid_of(rows * h), 256, 0, s>>>(R.att, rows, (int)kv, W.wo, W.bo, (int)h, R.x);
        rs_layernorm<<<ln_grid, 256, 0, s>>>(R.x, R.xn, rows, (int)h);
        rs_linear<RS_GELU><<<grid_of(rows * 4 * h), 256, 0, s>>>(R.xn, rows, (int)h, W.w1, W.b1, (int)(4 * h), R.h1);
        rs_linear<RS_RESID><<<grid_of(rows * h), 256, 0, s>>>(R.h1, rows, (int)(4 * h), W.w2, W.b2, (int)h, R.x);
    }
    // language_final_ln over every row, then each lane's last row (ReadSlice)
    rs_layernorm<<<ln_grid, 256, 0, s>>>(R.x, R.xn, rows, (int)h);
    rs_last_rows<<<grid_of(L * h), 256, 0, s>>>(R.xn, n, L, (int)h, R.last);
    rs_linear<RS_PLAIN><<<grid_of(L * V), 256, 0, s>>>(R.last, L, (int)h, R.lm_w, R.lm_b, (int)V, R.logits);
    check_launch();
}

}  // namespace

void reasoning_release(Ctx& c) {
    Reasoner& R = c.rs;
    if (R.step) cudaGraphExecDestroy(R.step);
    R.step = nullptr;
    if (R.h_ids) cudaFreeHost(R.h_ids);
    if (R.h_logits) cudaFreeHost(R.h_logits);
    R.h_ids = nullptr;
    R.h_logits = nullptr;
    for (void* p : R.bufs) c.dfree(p);
    R.bufs.clear();
    R.kv = nullptr;
    R.kv32 = nullptr;
    R.pos = nullptr;
    R.open = false;
    R.len = R.T = 0;
}

void reasoning_begin(Ctx& c, int64_t lanes, int64_t capacity) {
    const alpa_model_cfg& m = c.cfg;
    if (lanes < 1) fail(ALPA_ERR_CONFIG, "reasoning: lanes must be >= 1");
    if (capacity < 1) fail(ALPA_ERR_CONFIG, "reasoning: capacity must be >= 1");
    ensure_lm_weights(c);
    Reasoner& R = c.rs;
    // the KV buffer may still be the bound action prefix of an earlier scene
    if (c.prefix && c.prefix == R.kv) {
        c.prefix = nullptr;
        c.prefix_n = c.prefix_r = c.prefix_cap = 0;
        c.tm_pre_valid = false;
        invalidate_graph(c);
    }
    reasoning_release(c);
    const int64_t B = m.decoder_blocks, kv = m.kv_dim, h = m.hidden_dim;
    R.lanes = lanes;
    R.cap = capacity;
    const size_t kv_elems = (size_t)lanes * B * 2 * capacity * kv;
    R.kv = c.dalloc(kv_elems * c.esz());
    R.bufs.push_back(R.kv);
    ALPA_CUDA(cudaMemsetAsync(R.kv, 0, kv_elems * c.esz(), c.stream));
    if (c.bf16()) {
        R.kv32 = (float*)c.dalloc(kv_elems * sizeof(float));
        R.bufs.push_back(R.kv32);
    }
    // the position table covers every position a token can take (pipeline.cpp:291-295),
    // computed in double and rounded once, like sinusoidal_table (model.cpp:56-68)
    std::vector<float> pos((size_t)(capacity + 1) * h);
    for (int64_t p = 0; p <= capacity; ++p)
        for (int64_t i = 0; i < h; ++i) {
            const double e = static_cast<double>(2 * (i / 2)) / (double)h;
            const double ang = static_cast<double>(p) / std::pow(10000.0, e);
            pos[(size_t)p * h + i] = static_cast<float>((i % 2 == 0) ? std::sin(ang) : std::cos(ang));
        }
    R.pos = (float*)c.dalloc(pos.size() * sizeof(float));
    R.bufs.push_back(R.pos);
    ALPA_CUDA(cudaMemcpyAsync(R.pos, pos.data(), pos.size() * sizeof(float), cudaMemcpyHostToDevice, c.stream));
    R.dlen = (int64_t*)c.dalloc(sizeof(int64_t));
    R.bufs.push_back(R.dlen);
    ALPA_CUDA(cudaMallocHost(&R.h_ids, (size_t)lanes * sizeof(int32_t)));
    ALPA_CUDA(cudaMallocHost(&R.h_logits, (size_t)lanes * m.vocab_size * sizeof(float)));
    R.last = (float*)c.dalloc((size_t)lanes * h * sizeof(float));
    R.logits = (float*)c.dalloc((size_t)lanes * m.vocab_size * sizeof(float));
    R.bufs.push_back(R.last);
    R.bufs.push_back(R.logits);
    ALPA_CUDA(cudaStreamSynchronize(c.stream));
    R.open = true;
}

void reasoning_prefill(Ctx& c, const float* vision_rows, int64_t P, const int64_t* prompt_ids,
                       int64_t n_prompt, float* logits_out) {
    Reasoner& R = c.rs;
    if (!R.open) fail(ALPA_ERR_INTERNAL, "reasoning: not begun (or already sealed)");
    if (R.len != 0) fail(ALPA_ERR_INTERNAL, "prefill requires an empty, unsealed kv cache");
    const int64_t T = P + n_prompt;
    if (T < 1) fail(ALPA_ERR_INTERNAL, "prefill: need at least one token");
    if (T > R.cap) fail(ALPA_ERR_INTERNAL, "kv cache: reasoning capacity exceeded");
    if (P > 0 && !vision_rows) fail(ALPA_ERR_CONFIG, "null vision rows");
    if (n_prompt > 0 && !prompt_ids) fail(ALPA_ERR_CONFIG, "null prompt ids");
    const int64_t h = c.cfg.hidden_dim, V = c.cfg.vocab_size, L = R.lanes;
    for (int64_t i = 0; i < n_prompt; ++i)
        if (prompt_ids[i] < 0 || prompt_ids[i] >= V) fail(ALPA_ERR_CONFIG, "token id out of range");
    ensure_rows(c, L * T);
    cudaStream_t s = c.stream;
    // ctx = [vision rows | prompt embeddings] + pos, every lane (pipeline.cpp:297-324);
    // the caller's vision rows are [lanes][P][h] (the vision encoder output)
    float* vis = nullptr;
    if (P > 0) {
        vis = (float*)c.io((size_t)L * P * h * sizeof(float));  // context scratch, reused
        ALPA_CUDA(cudaMemcpyAsync(vis, vision_rows, (size_t)L * P * h * sizeof(float), cudaMemcpyHostToDevice, s));
    }
    if (n_prompt > 0) {
        ensure_ids(c, n_prompt);
        std::vector<int32_t> ids(prompt_ids, prompt_ids + n_prompt);
        ALPA_CUDA(cudaMemcpyAsync(R.ids, ids.data(), n_prompt * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    }
    for (int64_t l = 0; l < L; ++l) {
        if (P > 0)
            rs_embed_rows<<<grid_of(P * h), 256, 0, s>>>(nullptr, nullptr, vis + l * P * h, R.pos, P, (int)h, 0, 1,
                                                          h, l * T * h, R.x, nullptr);
        if (n_prompt > 0)
            rs_embed_rows<<<grid_of(n_prompt * h), 256, 0, s>>>(R.embed, R.ids, nullptr, R.pos, n_prompt, (int)h, P,
                                                                 1, h, (l * T + P) * h, R.x, nullptr);
    }
    check_launch();
    lm_forward(c, T, 0, nullptr);
    if (logits_out)
        ALPA_CUDA(cudaMemcpyAsync(logits_out, R.logits, (size_t)L * c.cfg.vocab_size * sizeof(float),
                                  cudaMemcpyDeviceToHost, s));
    // the device cache length the captured decode step reads
    ALPA_CUDA(cudaMemcpyAsync(R.dlen, &T, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    ALPA_CUDA(cudaStreamSynchronize(s));
    R.T = T;
    R.len = T;
}

void reasoning_decode(Ctx& c, const int64_t* ids, float* logits_out) {
    Reasoner& R = c.rs;
    if (!R.open || R.len == 0) fail(ALPA_ERR_INTERNAL, "reasoning: decode before prefill");
    if (R.len + 1 > R.cap) fail(ALPA_ERR_INTERNAL, "decode workspace too small for cache length");
    if (!ids) fail(ALPA_ERR_CONFIG, "null token ids");
    const int64_t h = c.cfg.hidden_dim, V = c.cfg.vocab_size, L = R.lanes;
    for (int64_t l = 0; l < L; ++l) {
        if (ids[l] < 0 || ids[l] >= V) fail(ALPA_ERR_CONFIG, "token id out of range");
        R.h_ids[l] = (int32_t)ids[l];
    }
    cudaStream_t s = c.stream;
    if (!R.step) {
        // One decode step (pipeline.cpp:371-386 + Model::decode_step + logits_head)
        // captured once per begin and replayed per token: the ids come from a
        // pinned host slot, the position (the cache length) from the device, and
        // the step ends by advancing it -- one graph launch per token.
        ensure_rows(c, L);
        ensure_ids(c, L);
        cudaGraph_t g = nullptr;
        ALPA_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        ALPA_CUDA(cudaMemcpyAsync(R.ids, R.h_ids, L * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        // x = embed(id) + pos[T + m - 1]: every lane's token sits at the next free row
        rs_embed_rows<<<grid_of(L * h), 256, 0, s>>>(R.embed, R.ids, nullptr, R.pos, L, (int)h, 0, 0, h, 0, R.x,
                                                      R.dlen);
        lm_forward(c, 1, 0, R.dlen);
        rs_bump<<<1, 32, 0, s>>>(R.dlen, 1);
        ALPA_CUDA(cudaMemcpyAsync(R.h_logits, R.logits, (size_t)L * V * sizeof(float), cudaMemcpyDeviceToHost, s));
        ALPA_CUDA(cudaStreamEndCapture(s, &g));
        ALPA_CUDA(cudaGraphInstantiate(&R.step, g, 0));
        cudaGraphDestroy(g);
    }
    ALPA_CUDA(cudaGraphLaunch(R.step, s));
    ALPA_CUDA(cudaStreamSynchronize(s));
    if (logits_out) std::memcpy(logits_out, R.h_logits, (size_t)L * V * sizeof(float));
    R.len += 1;
}

int64_t reasoning_seal(Ctx& c) {
    Reasoner& R = c.rs;
    if (!R.open) fail(ALPA_ERR_INTERNAL, "reasoning: nothing to seal");
    if (R.len < 1) fail(ALPA_ERR_INTERNAL, "kv cache: sealing an empty reasoning region");
    // KvCache::seal_reasoning: the produced K/V become the action stage's
    // prefix in place -- r live tokens inside the static capacity, no copy
    if (c.prefix && c.own_prefix) c.dfree(c.prefix);
    c.prefix = R.kv;
    c.own_prefix = false;  // owned by the reasoner (released by the next begin / destroy)
    c.prefix_n = R.lanes;
    c.prefix_r = R.len;
    c.prefix_cap = R.cap;
    refresh_prefix_map(c);
    invalidate_graph(c);
    R.open = false;
    return R.len;
}

}  // namespace alpa
