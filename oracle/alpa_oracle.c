/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle (checker) for the action-generation
 * hot path.  See alpa_oracle.h.  Compiled with -ffp-contract=off: every
 * multiply and add below rounds exactly as the reference's f32 code does.
 *
 * Reference anchors (all under /root/reference/proj):
 *   Rng                 include/minivla/common.hpp:36-59, src/common.cpp:48-55
 *   Fnv1a               include/minivla/common.hpp:63-76
 *   weight draw order   src/model.cpp:72-101, 120-151
 *   sinusoidal_table    src/model.cpp:56-68
 *   kernels             src/kernels_serial.cpp:11-93, include/minivla/kernels.hpp:60-72
 *   encode/decode/update src/model.cpp:555-598, attention src/model.cpp:280-324
 *   diffusion loop      src/model.cpp:607-636
 *   noise               src/pipeline.cpp:415-424
 *   rollout             src/pipeline.cpp:124-156
 */
#include "alpa_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ rng */

uint64_t orc_splitmix_next(uint64_t* s) {
    /* common.hpp:41-46 */
    uint64_t z = (*s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

float orc_next_float(uint64_t* s) {
    /* common.hpp:48-50 */
    return (float)(orc_splitmix_next(s) >> 40) * (1.0f / 16777216.0f);
}

float orc_uniform(uint64_t* s, float lo, float hi) {
    /* common.hpp:52 */
    return lo + (hi - lo) * orc_next_float(s);
}

float orc_normal(uint64_t* s) {
    /* common.cpp:48-55 */
    float u1 = orc_next_float(s);
    float u2 = orc_next_float(s);
    if (u1 < 1e-12f) u1 = 1e-12f;
    const float r = sqrtf(-2.0f * logf(u1));
    return r * cosf(6.28318530717958647692f * u2);
}

uint64_t orc_fnv1a(const void* data, int64_t n) {
    /* common.hpp:63-76 */
    const unsigned char* p = (const unsigned char*)data;
    uint64_t h = 0xcbf29ce484222325ULL;
    for (int64_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* -------------------------------------------------------------- weights */

static int64_t lin_count(int64_t in, int64_t out) { return in * out + out; }

static int64_t blk_count(int64_t w, int64_t kv) {
    /* draw_block, model.cpp:90-101: q,k,v [w->kv], o [kv->w], mlp1, mlp2 */
    return 3 * lin_count(w, kv) + lin_count(kv, w) + lin_count(w, 4 * w) +
           lin_count(4 * w, w);
}

int64_t orc_action_stream_offset(const orc_cfg* c) {
    /* model.cpp:125-139: patch_proj, vision blocks, token_embed, language
     * blocks, lm_head (norms draw nothing, model.cpp:83-88) */
    const int64_t patch_dim = c->patch_size * c->patch_size * 3;
    return lin_count(patch_dim, c->hidden_dim) +
           c->vision_blocks * blk_count(c->hidden_dim, c->kv_dim) +
           c->vocab_size * c->hidden_dim +
           c->decoder_blocks * blk_count(c->hidden_dim, c->kv_dim) +
           lin_count(c->hidden_dim, c->vocab_size);
}

int64_t orc_action_param_count(const orc_cfg* c) {
    const int64_t ah = c->action_hidden_dim;
    return lin_count(2, ah) + lin_count(ah, 4 * ah) + lin_count(4 * ah, ah) +
           c->decoder_blocks * blk_count(ah, c->kv_dim) + lin_count(ah, 2);
}

int orc_weights_build(const orc_cfg* c, orc_weights* w) {
    memset(w, 0, sizeof(*w));
    const int64_t ah = c->action_hidden_dim, kv = c->kv_dim, B = c->decoder_blocks;
    w->count = orc_action_param_count(c);
    w->arena = (float*)malloc((size_t)w->count * sizeof(float));
    w->blocks = (orc_linear*)calloc((size_t)(B * 6), sizeof(orc_linear));
    if (!w->arena || !w->blocks) return 3;
    /* splitmix is counter based: the k-th draw (0-based) sees state
     * seed + (k+1)*gamma, so jumping over the vision/language draws is O(1). */
    uint64_t state = c->weight_seed + (uint64_t)orc_action_stream_offset(c) *
                                          0x9e3779b97f4a7c15ULL;
    float* p = w->arena;
    const int64_t total = w->count;
    for (int64_t i = 0; i < total; ++i) p[i] = orc_uniform(&state, -0.05f, 0.05f);
    /* carve in draw order: w then b for each linear (draw_linear, model.cpp:72-81) */
#define CARVE(L, IN, OUT)                                                              \
    do {                                                                               \
        (L).in = (IN); (L).out = (OUT); (L).w = p; p += (IN) * (OUT); (L).b = p;        \
        p += (OUT);                                                                    \
    } while (0)
    CARVE(w->action_in, 2, ah);
    CARVE(w->mlp1, ah, 4 * ah);
    CARVE(w->mlp2, 4 * ah, ah);
    for (int64_t b = 0; b < B; ++b) {
        orc_linear* L = w->blocks + b * 6;
        CARVE(L[0], ah, kv);
        CARVE(L[1], ah, kv);
        CARVE(L[2], ah, kv);
        CARVE(L[3], kv, ah);
        CARVE(L[4], ah, 4 * ah);
        CARVE(L[5], 4 * ah, ah);
    }
    CARVE(w->head, ah, 2);
#undef CARVE
    return p == w->arena + total ? 0 : 3;
}

void orc_weights_free(orc_weights* w) {
    free(w->arena);
    free(w->blocks);
    memset(w, 0, sizeof(*w));
}

void orc_sinusoidal_table(int64_t positions, int64_t dim, float* table) {
    /* model.cpp:56-68 (double, then cast) */
    for (int64_t p = 0; p < positions; ++p) {
        for (int64_t i = 0; i < dim; ++i) {
            const double exponent = (double)(2 * (i / 2)) / (double)dim;
            const double freq = pow(10000.0, exponent);
            const double angle = (double)p / freq;
            table[p * dim + i] = (float)((i % 2 == 0) ? sin(angle) : cos(angle));
        }
    }
}

void orc_noise(uint64_t seed, uint64_t stride, int64_t lane0, int64_t n, int64_t steps,
               float* out) {
    /* pipeline.cpp:415-424 */
    for (int64_t l = 0; l < n; ++l) {
        uint64_t s = seed + (uint64_t)(lane0 + l) * stride;
        for (int64_t i = 0; i < steps * 2; ++i) out[l * steps * 2 + i] = orc_normal(&s);
    }
}

void orc_synthetic_prefix(uint64_t seed, int64_t blocks, int64_t r, int64_t kv,
                          float* out) {
    /* test_model.cpp:52-70 with lanes = 1 */
    for (int64_t b = 0; b < blocks; ++b) {
        uint64_t s = seed + (uint64_t)b;
        float* k = out + (b * 2) * r * kv;
        float* v = out + (b * 2 + 1) * r * kv;
        for (int64_t i = 0; i < r * kv; ++i) k[i] = orc_uniform(&s, -0.5f, 0.5f);
        for (int64_t i = 0; i < r * kv; ++i) v[i] = -k[i];
    }
}

/* --------------------------------------------------------------- kernels */

/* out[i][j] = sum_k a[i][k]*b[k][j], ascending k, f32 accumulator
 * (kernels_serial.cpp:11-26, kernels.hpp:60-72).  The loop nest is reordered
 * for cache reuse but each element sees exactly the reference's sequence of
 * roundings: acc=0; acc += a[k]*b[k][j] for k = 0..K-1. */
static void matmul_rows(const float* a, int64_t rows, int64_t K, const float* b,
                        int64_t N, float* out) {
    /* 16 x 256 output blocks: the weight rows are re-read rows/16 times instead
     * of rows/4 (the config-2 fixtures run the full 36-block depth) */
    const int64_t nib = (rows + 15) / 16, njb = (N + 255) / 256;
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
    for (int64_t ib = 0; ib < nib; ++ib) {
        for (int64_t jb = 0; jb < njb; ++jb) {
            const int64_t i0 = ib * 16, j0 = jb * 256;
            const int64_t ni = rows - i0 < 16 ? rows - i0 : 16;
            const int64_t nj = N - j0 < 256 ? N - j0 : 256;
            float acc[16][256];
            for (int64_t r = 0; r < ni; ++r)
                for (int64_t j = 0; j < nj; ++j) acc[r][j] = 0.0f;
            for (int64_t k = 0; k < K; ++k) {
                const float* brow = b + k * N + j0;
                for (int64_t r = 0; r < ni; ++r) {
                    const float av = a[(i0 + r) * K + k];
                    for (int64_t j = 0; j < nj; ++j) acc[r][j] += av * brow[j];
                }
            }
            for (int64_t r = 0; r < ni; ++r)
                memcpy(out + (i0 + r) * N + j0, acc[r], (size_t)nj * sizeof(float));
        }
    }
}

/* emit_linear (model.cpp:209-226): matmul then a separate broadcast bias add
 * (add_row, kernels_serial.cpp:28-33). */
static void linear(const float* x, int64_t rows, const orc_linear* L, float* out) {
    matmul_rows(x, rows, L->in, L->w, L->out, out);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < L->out; ++j) out[i * L->out + j] = out[i * L->out + j] + L->b[j];
}

static void add_inplace(float* a, const float* b, int64_t count) {
    /* add_row with b of equal shape */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; ++i) a[i] = a[i] + b[i];
}

static void layernorm(const float* x, int64_t rows, int64_t n, float* out) {
    /* layernorm_row, kernels_serial.cpp:66-84, gamma=1 beta=0
     * (make_norm, model.cpp:83-88), eps=1e-5 (substrate.hpp:56) */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) {
        const float* xr = x + i * n;
        float* o = out + i * n;
        float mean = 0.0f;
        for (int64_t j = 0; j < n; ++j) mean += xr[j];
        mean /= (float)n;
        float var = 0.0f;
        for (int64_t j = 0; j < n; ++j) {
            const float d = xr[j] - mean;
            var += d * d;
        }
        var /= (float)n;
        const float inv = 1.0f / sqrtf(var + 1e-5f);
        for (int64_t j = 0; j < n; ++j) o[j] = (xr[j] - mean) * inv * 1.0f + 0.0f;
    }
}

static void gelu_inplace(float* a, int64_t count) {
    /* gelu_row, kernels_serial.cpp:86-93 */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; ++i) {
        const float x = a[i];
        a[i] = 0.5f * x * (1.0f + erff(x * 0.70710678118654752440f));
    }
}

/* emit_attention (model.cpp:280-324) over the attend_view of one block
 * (kv_cache.cpp:247-263): lane l sees [prefix(l) rows 0..r-1 || its own 64
 * action rows].  Scores = alpha*dot (alpha applied after the dot,
 * kernels_serial.cpp:24), softmax_row (kernels_serial.cpp:41-64, non-causal),
 * ctx = P.V with ascending-token accumulation (dot_col). */
static void attention(const orc_cfg* c, const float* q, const float* pk, const float* pv,
                      int64_t prefix_lane_stride, const int32_t* lane_prefix,
                      int64_t r, const float* ak, const float* av, int64_t n,
                      float* ctx) {
    const int64_t kd = c->kv_dim, H = c->heads, hd = kd / H, A = c->action_steps;
    const int64_t T = r + A;
    const float alpha = 1.0f / sqrtf((float)hd);
#pragma omp parallel
    {
        float* s = (float*)malloc((size_t)T * sizeof(float));
#pragma omp for collapse(3) schedule(static)
        for (int64_t l = 0; l < n; ++l) {
            for (int64_t h = 0; h < H; ++h) {
                for (int64_t i = 0; i < A; ++i) {
                    const int64_t pl = lane_prefix ? lane_prefix[l] : 0;
                    const float* kbase = pk + pl * prefix_lane_stride;
                    const float* vbase = pv + pl * prefix_lane_stride;
                    const float* qr = q + (l * A + i) * kd + h * hd;
                    for (int64_t j = 0; j < T; ++j) {
                        const float* kr = j < r ? kbase + j * kd + h * hd
                                                : ak + (l * A + (j - r)) * kd + h * hd;
                        float acc = 0.0f;
                        for (int64_t d = 0; d < hd; ++d) acc += qr[d] * kr[d];
                        s[j] = alpha * acc;
                    }
                    float mx = s[0];
                    for (int64_t j = 1; j < T; ++j)
                        if (s[j] > mx) mx = s[j];
                    float sum = 0.0f;
                    for (int64_t j = 0; j < T; ++j) {
                        const float e = expf(s[j] - mx);
                        s[j] = e;
                        sum += e;
                    }
                    const float inv = 1.0f / sum;
                    for (int64_t j = 0; j < T; ++j) s[j] *= inv;
                    /* dot_col per output dim d, ascending j.  Loop nest reordered
                     * (j outer, d inner, one accumulator per d): every element
                     * still sees acc=0; acc += s[j]*v[j][d] for j = 0..T-1. */
                    float* o = ctx + (l * A + i) * kd + h * hd;
                    for (int64_t d = 0; d < hd; ++d) o[d] = 0.0f;
                    for (int64_t j = 0; j < T; ++j) {
                        const float* vr = j < r ? vbase + j * kd + h * hd
                                                : av + (l * A + (j - r)) * kd + h * hd;
                        const float sj = s[j];
                        for (int64_t d = 0; d < hd; ++d) o[d] += sj * vr[d];
                    }
                }
            }
        }
        free(s);
    }
}

int orc_diffusion_refine(const orc_cfg* c, const orc_weights* w, const float* prefix,
                         int64_t r, const int32_t* lane_prefix, int64_t n, int64_t iters,
                         float* actions, int threads) {
#ifdef _OPENMP
    const int saved = omp_get_max_threads();
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
    const int64_t ah = c->action_hidden_dim, kd = c->kv_dim, A = c->action_steps;
    const int64_t B = c->decoder_blocks, M = n * A;
    float* pos = (float*)malloc((size_t)(A * ah) * sizeof(float));
    float* e0 = (float*)malloc((size_t)(M * ah) * sizeof(float));
    float* e = (float*)malloc((size_t)(M * ah) * sizeof(float));
    float* xn = (float*)malloc((size_t)(M * ah) * sizeof(float));
    float* tmp = (float*)malloc((size_t)(M * ah) * sizeof(float));
    float* h1 = (float*)malloc((size_t)(M * 4 * ah) * sizeof(float));
    float* q = (float*)malloc((size_t)(M * kd) * sizeof(float));
    float* k = (float*)malloc((size_t)(M * kd) * sizeof(float));
    float* v = (float*)malloc((size_t)(M * kd) * sizeof(float));
    float* ctx = (float*)malloc((size_t)(M * kd) * sizeof(float));
    float* delta = (float*)malloc((size_t)(M * 2) * sizeof(float));
    int rc = 0;
    if (!pos || !e0 || !e || !xn || !tmp || !h1 || !q || !k || !v || !ctx || !delta) {
        rc = 3;
        goto done;
    }
    /* make_action_workspace: the [64][ah] table tiled over lanes (model.cpp:531-538) */
    orc_sinusoidal_table(A, ah, pos);
    const int64_t prefix_lane_stride = B * 2 * r * kd; /* [lane][B][2][r][kv] when multi */
    for (int64_t it = 1; it <= iters; ++it) {
        /* emit_action_encode, model.cpp:555-563 */
        linear(actions, M, &w->action_in, e0);
        for (int64_t i = 0; i < M; ++i)
            for (int64_t j = 0; j < ah; ++j)
                e0[i * ah + j] = e0[i * ah + j] + pos[(i % A) * ah + j];
        linear(e0, M, &w->mlp1, h1);
        gelu_inplace(h1, M * 4 * ah);
        linear(h1, M, &w->mlp2, e);
        /* emit_action_decoder, model.cpp:565-592 */
        for (int64_t b = 0; b < B; ++b) {
            const orc_linear* L = w->blocks + b * 6;
            layernorm(e, M, ah, xn);
            linear(xn, M, &L[0], q);
            linear(xn, M, &L[1], k);
            linear(xn, M, &L[2], v);
            /* write_action_kv + attend_view: prefix rows then this lane's rows */
            const float* pk = prefix + (b * 2) * r * kd;
            const float* pv = prefix + (b * 2 + 1) * r * kd;
            attention(c, q, pk, pv, prefix_lane_stride, lane_prefix, r, k, v, n, ctx);
            linear(ctx, M, &L[3], tmp);
            add_inplace(e, tmp, M * ah);
            layernorm(e, M, ah, xn);
            linear(xn, M, &L[4], h1);
            gelu_inplace(h1, M * 4 * ah);
            linear(h1, M, &L[5], tmp);
            add_inplace(e, tmp, M * ah);
        }
        layernorm(e, M, ah, xn);
        linear(xn, M, &w->head, delta);
        /* emit_action_update, model.cpp:594-598: two separate roundings */
        for (int64_t i = 0; i < M * 2; ++i) {
            const float ds = c->update_scale * delta[i];
            actions[i] = actions[i] + ds;
        }
    }
done:
    free(pos); free(e0); free(e); free(xn); free(tmp); free(h1);
    free(q); free(k); free(v); free(ctx); free(delta);
#ifdef _OPENMP
    omp_set_num_threads(saved);
#endif
    return rc;
}

/* --------------------------------------------------------------- rollout */

int orc_rollout(const float* actions, int64_t n, int64_t steps, float v0, float* traj) {
    /* actions_to_trajectory, pipeline.cpp:124-148 */
    if (v0 < 0.0f || !isfinite(v0)) return 3;
    const double dt = 0.1;
    for (int64_t l = 0; l < n; ++l) {
        double x = 0.0, y = 0.0, yaw = 0.0, v = v0;
        for (int64_t i = 0; i < steps; ++i) {
            const float a = actions[(l * steps + i) * 2];
            const float k = actions[(l * steps + i) * 2 + 1];
            if (!isfinite(a) || !isfinite(k)) return 3;
            const double nx = x + v * cos(yaw) * dt;
            const double ny = y + v * sin(yaw) * dt;
            const double nyaw = yaw + (double)k * v * dt;
            const double nv = v + (double)a * dt;
            x = nx; y = ny; yaw = nyaw; v = nv;
            traj[(l * steps + i) * 3] = (float)x;
            traj[(l * steps + i) * 3 + 1] = (float)y;
            traj[(l * steps + i) * 3 + 2] = (float)yaw;
        }
    }
    return 0;
}

float orc_initial_speed(const float* h) {
    /* pipeline.cpp:150-156 */
    const double dx = (double)h[15 * 3] - (double)h[14 * 3];
    const double dy = (double)h[15 * 3 + 1] - (double)h[14 * 3 + 1];
    return (float)(sqrt(dx * dx + dy * dy) / 0.1);
}

int64_t orc_kv_footprint_bytes(int64_t blocks, int64_t batch, int64_t tokens,
                               int64_t kv_dim, int64_t elem_bytes) {
    return blocks * batch * tokens * kv_dim * 2 * elem_bytes;
}

/* --------------------------------------------------------------- open-loop metrics */

static double mean_displacement(const float* a, const float* b, int64_t steps) {
    /* eval.cpp:14-25: double accumulation in pose order (no FMA: -ffp-contract=off) */
    double sum = 0.0;
    for (int64_t i = 0; i < steps; ++i) {
        const double dx = (double)a[i * 3] - (double)b[i * 3];
        const double dy = (double)a[i * 3 + 1] - (double)b[i * 3 + 1];
        sum += sqrt(dx * dx + dy * dy);
    }
    return sum / (double)steps;
}

int orc_min_ade(const float* traj, int64_t n, int64_t steps, const float* gt, double* out) {
    /* eval.cpp:39-46 */
    if (n < 1) return 3;
    double best = mean_displacement(traj, gt, steps);
    for (int64_t i = 1; i < n; ++i) {
        const double d = mean_displacement(traj + i * steps * 3, gt, steps);
        best = d < best ? d : best; /* std::min(best, d) */
    }
    *out = best;
    return 0;
}

int orc_diversity(const float* traj, int64_t n, int64_t steps, double* out) {
    /* eval.cpp:48-59 */
    if (n < 2) return 3;
    double sum = 0.0;
    int64_t pairs = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = i + 1; j < n; ++j) {
            sum += mean_displacement(traj + i * steps * 3, traj + j * steps * 3, steps);
            pairs += 1;
        }
    *out = sum / (double)pairs;
    return 0;
}
