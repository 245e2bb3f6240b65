// Action-expert weights and the prefix KV, generated or uploaded into the
// device layouts the kernels want.
//
// Weight stream: ModelWeights::build (model.cpp:120-151) draws every tensor
// from ONE splitmix64 Rng(weight_seed) as uniform(-0.05, 0.05) in the order
// patch_proj, vision blocks, token_embed, language blocks, lm_head,
// action_in, action_mlp1, action_mlp2, action blocks (q,k,v,o,mlp1,mlp2; w
// [in][out] then b), action_head (draw_linear model.cpp:72-81, draw_block
// model.cpp:90-101).  The action tensors start at draw S = stream_offset();
// each device thread evaluates its own draw by jump-ahead (splitmix_at).
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "ctx.h"

namespace alpa {

static int64_t lin_count(int64_t in, int64_t out) { return in * out + out; }
static int64_t blk_count(int64_t w, int64_t kv) {
    return 3 * lin_count(w, kv) + lin_count(kv, w) + lin_count(w, 4 * w) + lin_count(4 * w, w);
}

int64_t stream_offset(const alpa_model_cfg& c) {
    const int64_t patch_dim = c.patch_size * c.patch_size * 3;
    return lin_count(patch_dim, c.hidden_dim) + c.vision_blocks * blk_count(c.hidden_dim, c.kv_dim) +
           c.vocab_size * c.hidden_dim + c.decoder_blocks * blk_count(c.hidden_dim, c.kv_dim) +
           lin_count(c.hidden_dim, c.vocab_size);
}

int64_t param_count(const alpa_model_cfg& c) {
    const int64_t ah = c.action_hidden_dim;
    return lin_count(2, ah) + lin_count(ah, 4 * ah) + lin_count(4 * ah, ah) +
           c.decoder_blocks * blk_count(ah, c.kv_dim) + lin_count(ah, 2);
}

namespace {

struct Src {
    const float* arena;  // host-uploaded arena (draw order) or nullptr
    uint64_t seed;
    int64_t offset;      // draw index of the arena's element 0
};

__device__ inline float draw(const Src& s, int64_t k) {
    return s.arena ? s.arena[k] : uniform_at(s.seed, (uint64_t)(s.offset + k), -0.05f, 0.05f);
}

// w element (i, j) of an [in][out] linear whose first draw is `base`.
// f32 layout:  dst[i*ld + col_off + j]            (reference [in][out])
// bf16 layout: dst[(col_off + j)*in + i]          (W^T, K-major for tcgen05)
__global__ void place_weight_f32(Src s, int64_t base, int64_t in, int64_t out, float* dst,
                                 int64_t ld, int64_t col_off) {
    const int64_t total = in * out;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / out, j = t % out;
        dst[i * ld + col_off + j] = draw(s, base + t);
    }
}

__global__ void place_weight_bf16t(Src s, int64_t base, int64_t in, int64_t out,
                                   __nv_bfloat16* dst, int64_t col_off) {
    const int64_t total = in * out;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / in, i = t % in;  // consecutive threads -> consecutive i
        dst[(col_off + j) * in + i] = __float2bfloat16_rn(draw(s, base + i * out + j));
    }
}

__global__ void place_bias(Src s, int64_t base, int64_t out, float* dst, int64_t off) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < out;
         j += (int64_t)gridDim.x * blockDim.x)
        dst[off + j] = draw(s, base + j);
}

// make_sealed_cache (tests/test_model.cpp:52-70), lane 0: per block Rng(seed+b),
// K token-major uniform(-0.5, 0.5), V = -K.  out [B][2][r][kv].
template <typename T>
__global__ void synth_prefix(uint64_t seed, int64_t blocks, int64_t r, int64_t kv, T* out) {
    const int64_t per = r * kv, total = blocks * per;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / per, i = t % per;
        const float k = uniform_at(seed + (uint64_t)b, (uint64_t)i, -0.5f, 0.5f);
        if constexpr (sizeof(T) == 2) {
            out[(b * 2) * per + i] = __float2bfloat16_rn(k);
            out[(b * 2 + 1) * per + i] = __float2bfloat16_rn(-k);
        } else {
            out[(b * 2) * per + i] = k;
            out[(b * 2 + 1) * per + i] = -k;
        }
    }
}

// colsum[f] = sum_k W^T[f][k] over the bf16-rounded weights (LN fold).
__global__ void row_sums_bf16(const __nv_bfloat16* __restrict__ w, int64_t rows, int64_t k,
                              float* __restrict__ out) {
    const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    float s = 0.f;
    for (int64_t j = lane; j < k; j += 32) s += __bfloat162float(w[row * k + j]);
    s = warp_sum(s);
    if (lane == 0) out[row] = s;
}

__global__ void f32_to_bf16(const float* in, __nv_bfloat16* out, int64_t n) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x)
        out[t] = __float2bfloat16_rn(in[t]);
}

inline int grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    return (int)(g > 148 * 32 ? 148 * 32 : (g < 1 ? 1 : g));
}

}  // namespace

void draw_linear_f32(Ctx& c, int64_t base, int64_t in, int64_t out, float* w, float* b) {
    Src src{nullptr, c.cfg.weight_seed, 0};
    place_weight_f32<<<grid_for(in * out), 256, 0, c.stream>>>(src, base, in, out, w, out, 0);
    place_bias<<<grid_for(out), 256, 0, c.stream>>>(src, base + in * out, out, b, 0);
    ALPA_CUDA(cudaGetLastError());
}

void draw_array_f32(Ctx& c, int64_t base, int64_t n, float* dst) {
    Src src{nullptr, c.cfg.weight_seed, 0};
    place_bias<<<grid_for(n), 256, 0, c.stream>>>(src, base, n, dst, 0);
    ALPA_CUDA(cudaGetLastError());
}

void load_weights(Ctx& c, const float* host_arena, int64_t count, uint64_t seed, int64_t offset) {
    const alpa_model_cfg& cfg = c.cfg;
    const int64_t ah = cfg.action_hidden_dim, kv = cfg.kv_dim, B = cfg.decoder_blocks;
    const int64_t total = param_count(cfg);
    if (host_arena && count != total)
        fail(ALPA_ERR_CONFIG, "weight arena has " + std::to_string(count) + " values, expected " +
                                  std::to_string(total));
    cudaStream_t s = c.stream;
    Src src{nullptr, seed, offset};
    float* staged = nullptr;
    if (host_arena) {
        ALPA_CUDA(cudaMalloc(&staged, total * sizeof(float)));
        ALPA_CUDA(cudaMemcpyAsync(staged, host_arena, total * sizeof(float), cudaMemcpyHostToDevice, s));
        src.arena = staged;
    }
    int64_t cursor = 0;  // draw index relative to action_in.w
    const bool bf = c.bf16();

    // f32 [in][out] linear (always f32: action_in K=2 and head N=2 are tiny
    // SIMT epilogue math on both paths).
    auto f32_linear = [&](Linear& L, int64_t in, int64_t out) {
        L.in = in; L.out = out;
        L.w = c.dalloc(in * out * sizeof(float));
        L.b = (float*)c.dalloc(out * sizeof(float));
        place_weight_f32<<<grid_for(in * out), 256, 0, s>>>(src, cursor, in, out, (float*)L.w, out, 0);
        place_bias<<<grid_for(out), 256, 0, s>>>(src, cursor + in * out, out, L.b, 0);
        cursor += in * out + out;
    };
    // GEMM operand: f32 [in][ld] or bf16 W^T [ld][in], written at column col_off
    auto gemm_linear = [&](Linear& L, int64_t in, int64_t out, int64_t col_off) {
        if (bf)
            place_weight_bf16t<<<grid_for(in * out), 256, 0, s>>>(src, cursor, in, out,
                                                                 (__nv_bfloat16*)L.w, col_off);
        else
            place_weight_f32<<<grid_for(in * out), 256, 0, s>>>(src, cursor, in, out, (float*)L.w,
                                                               L.out, col_off);
        place_bias<<<grid_for(out), 256, 0, s>>>(src, cursor + in * out, out, L.b, col_off);
        cursor += in * out + out;
    };
    auto alloc_gemm = [&](Linear& L, int64_t in, int64_t out) {
        L.in = in; L.out = out;
        L.w = c.dalloc(in * out * (bf ? 2 : 4));
        L.b = (float*)c.dalloc(out * sizeof(float));
    };

    f32_linear(c.act_in, 2, ah);
    alloc_gemm(c.mlp1, ah, 4 * ah);
    gemm_linear(c.mlp1, ah, 4 * ah, 0);
    alloc_gemm(c.mlp2, 4 * ah, ah);
    gemm_linear(c.mlp2, 4 * ah, ah, 0);
    c.blocks.assign(B, Block{});
    for (int64_t b = 0; b < B; ++b) {
        Block& blk = c.blocks[b];
        alloc_gemm(blk.qkv, ah, 3 * kv);
        gemm_linear(blk.qkv, ah, kv, 0);       // q
        gemm_linear(blk.qkv, ah, kv, kv);      // k
        gemm_linear(blk.qkv, ah, kv, 2 * kv);  // v
        alloc_gemm(blk.o, kv, ah);
        gemm_linear(blk.o, kv, ah, 0);
        alloc_gemm(blk.mlp1, ah, 4 * ah);
        gemm_linear(blk.mlp1, ah, 4 * ah, 0);
        alloc_gemm(blk.mlp2, 4 * ah, ah);
        gemm_linear(blk.mlp2, 4 * ah, ah, 0);
    }
    f32_linear(c.head, ah, 2);
    if (cursor != total) fail(ALPA_ERR_INTERNAL, "weight draw order mismatch");

    if (bf) {
        auto map = [&](Linear& L) {
            make_tmap_bf16_2d(&L.tmap, L.w, (uint64_t)L.in, (uint64_t)L.out, (uint64_t)L.in * 2, 64,
                              128);
        };
        map(c.mlp1);
        map(c.mlp2);
        auto colsum = [&](Linear& L) {
            L.colsum = (float*)c.dalloc(L.out * sizeof(float));
            row_sums_bf16<<<(unsigned)((L.out + 7) / 8), 256, 0, s>>>((const __nv_bfloat16*)L.w,
                                                                      L.out, L.in, L.colsum);
        };
        for (auto& blk : c.blocks) {
            map(blk.qkv); map(blk.o); map(blk.mlp1); map(blk.mlp2);
            colsum(blk.qkv);
            colsum(blk.mlp1);
        }
    }

    // sinusoidal_table (model.cpp:56-68), double then cast, host side as in
    // make_action_workspace (model.cpp:531-538).
    const int64_t A = cfg.action_steps;
    std::vector<float> table(A * ah);
    for (int64_t p = 0; p < A; ++p)
        for (int64_t i = 0; i < ah; ++i) {
            const double exponent = static_cast<double>(2 * (i / 2)) / static_cast<double>(ah);
            const double angle = static_cast<double>(p) / std::pow(10000.0, exponent);
            table[p * ah + i] = static_cast<float>((i % 2 == 0) ? std::sin(angle) : std::cos(angle));
        }
    c.pos = (float*)c.dalloc(A * ah * sizeof(float));
    ALPA_CUDA(cudaMemcpyAsync(c.pos, table.data(), A * ah * sizeof(float), cudaMemcpyHostToDevice, s));
    ALPA_CUDA(cudaGetLastError());
    ALPA_CUDA(cudaStreamSynchronize(s));
    if (staged) cudaFree(staged);
    c.weights_ready = true;
}

static void release_prefix(Ctx& c) {
    if (c.prefix && c.own_prefix) c.dfree(c.prefix);
    c.prefix = nullptr;
    c.own_prefix = false;
}

void synthesize_prefix_into(Ctx& c, void* dst, uint64_t seed, int64_t r) {
    if (r < 1) fail(ALPA_ERR_INTERNAL, "kv cache: sealing an empty reasoning region");
    const int64_t B = c.cfg.decoder_blocks, kv = c.cfg.kv_dim;
    if (c.bf16())
        synth_prefix<__nv_bfloat16><<<grid_for(B * r * kv), 256, 0, c.stream>>>(
            seed, B, r, kv, (__nv_bfloat16*)dst);
    else
        synth_prefix<float><<<grid_for(B * r * kv), 256, 0, c.stream>>>(seed, B, r, kv,
                                                                        (float*)dst);
    ALPA_CUDA(cudaGetLastError());
}

void make_prefix_synthetic(Ctx& c, uint64_t seed, int64_t r) {
    if (r < 1) fail(ALPA_ERR_INTERNAL, "kv cache: sealing an empty reasoning region");
    release_prefix(c);
    const int64_t n = c.cfg.decoder_blocks * 2 * r * c.cfg.kv_dim;
    c.prefix = c.dalloc(n * c.esz());
    c.own_prefix = true;
    synthesize_prefix_into(c, c.prefix, seed, r);
    ALPA_CUDA(cudaStreamSynchronize(c.stream));
    c.prefix_n = 1;
    c.prefix_r = r;
    c.prefix_cap = r;
    refresh_prefix_map(c);
}

void make_prefix_from_host(Ctx& c, const float* host, int64_t n_prefix, int64_t r) {
    if (r < 1) fail(ALPA_ERR_INTERNAL, "kv cache: sealing an empty reasoning region");
    if (n_prefix < 1) fail(ALPA_ERR_CONFIG, "prefix count must be >= 1");
    release_prefix(c);
    const int64_t n = n_prefix * c.cfg.decoder_blocks * 2 * r * c.cfg.kv_dim;
    c.prefix = c.dalloc(n * c.esz());
    c.own_prefix = true;
    if (c.bf16()) {
        float* staged = nullptr;
        ALPA_CUDA(cudaMalloc(&staged, n * sizeof(float)));
        ALPA_CUDA(cudaMemcpyAsync(staged, host, n * sizeof(float), cudaMemcpyHostToDevice, c.stream));
        f32_to_bf16<<<grid_for(n), 256, 0, c.stream>>>(staged, (__nv_bfloat16*)c.prefix, n);
        ALPA_CUDA(cudaStreamSynchronize(c.stream));
        cudaFree(staged);
    } else {
        ALPA_CUDA(cudaMemcpyAsync(c.prefix, host, n * sizeof(float), cudaMemcpyHostToDevice, c.stream));
        ALPA_CUDA(cudaStreamSynchronize(c.stream));
    }
    c.prefix_n = n_prefix;
    c.prefix_r = r;
    c.prefix_cap = r;
    refresh_prefix_map(c);
}

}  // namespace alpa
