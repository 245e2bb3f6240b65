/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle (checker) for the action-generation
 * hot path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product library never links it.
 *
 * Plain-C restatement of the reference's f32 path
 * (/root/reference/proj, "minivla"): every function cites the reference
 * file:line it restates.  Built with -ffp-contract=off so the arithmetic is
 * the reference's canonical bits.  Parity is pinned against
 * the reference itself (oracle/_ref/libminivla_ref.so, compiled from the
 * reference sources by oracle/Makefile) and against the golden digests in
 * tests/golden/ (see tests/test_oracle.py).
 */
#ifndef ALPA_ORACLE_H
#define ALPA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors ModelConfig (include/minivla/model.hpp:12-29). */
typedef struct orc_cfg {
    int64_t vision_blocks;
    int64_t decoder_blocks;
    int64_t hidden_dim;
    int64_t action_hidden_dim;
    int64_t kv_dim;
    int64_t heads;
    int64_t vocab_size;
    int64_t patch_size;
    int64_t action_steps;
    int64_t diffusion_iters;
    int64_t max_new_tokens;
    float update_scale;
    uint64_t weight_seed;
} orc_cfg;

/* ---- common.hpp:36-59 / common.cpp:48-55 (splitmix64 Rng) ---- */
uint64_t orc_splitmix_next(uint64_t* state);
float orc_next_float(uint64_t* state);
float orc_uniform(uint64_t* state, float lo, float hi);
float orc_normal(uint64_t* state);

/* ---- common.hpp:63-76 (Fnv1a) ---- */
uint64_t orc_fnv1a(const void* data, int64_t n);

/* Number of uniform draws ModelWeights::build consumes before action_in
 * (model.cpp:120-140). */
int64_t orc_action_stream_offset(const orc_cfg* c);
/* Total action-expert parameter count (model.cpp:141-149). */
int64_t orc_action_param_count(const orc_cfg* c);

/* Action-expert weights in the reference layout: w [in][out] row-major,
 * b [out] (model.hpp:54-59).  One contiguous float arena; tensors in draw order
 * (model.cpp:141-149): action_in, mlp1, mlp2, blocks (q,k,v,o,mlp1,mlp2), head. */
typedef struct orc_linear { const float* w; const float* b; int64_t in, out; } orc_linear;
typedef struct orc_weights {
    float* arena;
    int64_t count;
    orc_linear action_in, mlp1, mlp2, head;
    orc_linear* blocks; /* decoder_blocks * 6: q,k,v,o,mlp1,mlp2 */
} orc_weights;

int orc_weights_build(const orc_cfg* c, orc_weights* w);
void orc_weights_free(orc_weights* w);

/* sinusoidal_table (model.cpp:56-68): [positions][dim]. */
void orc_sinusoidal_table(int64_t positions, int64_t dim, float* out);

/* Host noise (pipeline.cpp:415-424): lanes [lane0, lane0+n), 128 normals each,
 * lane l seeded with seed + l*stride.  out [n][64][2]. */
void orc_noise(uint64_t seed, uint64_t stride, int64_t lane0, int64_t n,
               int64_t steps, float* out);

/* make_sealed_cache recipe (tests/test_model.cpp:43-74), batch 1:
 * per block Rng(seed+b), K uniform(-0.5,0.5) token-major, V = -K.
 * out [B][2][r][kv]. */
void orc_synthetic_prefix(uint64_t seed, int64_t blocks, int64_t r, int64_t kv,
                          float* out);

/* Model::diffusion_refine (model.cpp:607-636) with every op of
 * emit_action_encode/decoder/update (model.cpp:555-598) and emit_attention
 * (model.cpp:280-324) in the reference's order.
 *   prefix      [B][2][r][kv] f32, shared by every lane when lane_prefix==NULL;
 *               otherwise prefix has n_prefix entries and lane l uses
 *               lane_prefix[l] (multi topology).
 *   actions     [n][64][2] in/out.
 *   iters       K (the reference uses ModelConfig::diffusion_iters).
 *   threads     OpenMP threads (<=0: runtime default). */
int orc_diffusion_refine(const orc_cfg* c, const orc_weights* w, const float* prefix,
                         int64_t r, const int32_t* lane_prefix, int64_t n,
                         int64_t iters, float* actions, int threads);

/* actions_to_trajectory (pipeline.cpp:124-148): [n][64][2] -> [n][64][3].
 * Returns 3 (InternalError) on bad speed / non-finite actions. */
int orc_rollout(const float* actions, int64_t n, int64_t steps, float v0, float* traj);

/* Open-loop metrics (eval.cpp:14-59): trajectories traj [n][steps][3] (x, y, yaw;
 * only x, y used), ground truth gt [steps][3].  mean_displacement is the mean of
 * sqrt(dx^2 + dy^2) over the poses in double, summed in pose order
 * (eval.cpp:14-25); min_ade = min over samples in sample order (eval.cpp:39-46);
 * diversity = mean over pairs i < j in row-major pair order (eval.cpp:48-59).
 * Return 3 (InternalError) for n < 1 (min_ade) / n < 2 (diversity). */
int orc_min_ade(const float* traj, int64_t n, int64_t steps, const float* gt, double* out);
int orc_diversity(const float* traj, int64_t n, int64_t steps, double* out);

/* initial_speed_from_history (pipeline.cpp:150-156); history [16][3]. */
float orc_initial_speed(const float* history);

/* kv_footprint_bytes (kv_cache.cpp:22-26). */
int64_t orc_kv_footprint_bytes(int64_t blocks, int64_t batch, int64_t tokens,
                               int64_t kv_dim, int64_t elem_bytes);

#ifdef __cplusplus
}
#endif
#endif
