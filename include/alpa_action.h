/*
 * alpa_action.h — C-ABI of the B200-native action-generation hot path.
 *
 * Drop-in boundary for the reference's single-reasoning action generation
 * (arXiv 2605.08975 reference "minivla", /root/reference/proj):
 *
 *   reference                                              replaced by
 *   ---------------------------------------------------------------------------
 *   Engine::run_action_generation   pipeline.hpp:145-148   alpa_generate
 *     (replicate_for_batch kv_cache.cpp:280-318, host noise pipeline.cpp:415-424,
 *      diffusion_refine model.cpp:607-636, read_actions model.cpp:638-650)
 *   actions_to_trajectory           pipeline.hpp:90         fused into alpa_generate
 *                                                           (traj_out), alpa_rollout
 *   initial_speed_from_history      pipeline.hpp:93         alpa_initial_speed
 *   ModelWeights::build + Model::Model model.cpp:120-207    alpa_load_weights_seeded /
 *                                                           alpa_load_weights_host
 *   ReasoningOutput::kv (sealed KvCache, pipeline.hpp:120)  alpa_bind_prefix*
 *   kv_footprint_bytes              kv_cache.hpp:26-28      alpa_kv_footprint_bytes
 *   Error taxonomy                  common.hpp:10-23        ALPA_ERR_* + alpa_last_error
 *
 * Plain pointers and sizes only.  Host buffers are caller-owned; device state
 * (weights, the single prefix copy, workspaces, the captured CUDA graph) is
 * owned by the context.  One context = one CUDA stream + its graphs; not
 * thread-safe (Substrate single-owner contract, substrate.hpp:114-115);
 * distinct contexts are independent.  See INTEGRATION.md for the C++ shim
 * that re-exposes the reference signature.
 */
#ifndef ALPA_ACTION_H
#define ALPA_ACTION_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes mirror the reference's exit-code taxonomy (common.hpp:10-11,
 * cli.cpp:528-540): IoError -> 1, ConfigError -> 2, InternalError -> 3. */
#define ALPA_OK 0
#define ALPA_ERR_IO 1
#define ALPA_ERR_CONFIG 2
#define ALPA_ERR_INTERNAL 3

/* Arithmetic of the denoising loop. */
#define ALPA_DTYPE_F32 0  /* fp32 SIMT path: parity bar rel-L2 <= 1e-4         */
#define ALPA_DTYPE_BF16 1 /* bf16 operands on tcgen05, fp32 accumulate/residual/
                             softmax/LN stats: parity bar rel-L2 <= 2e-2        */

/* KvStrategy (kv_cache.hpp:9) and ExecMode (model.hpp:43). */
#define ALPA_KV_DYNAMIC 0
#define ALPA_KV_STATIC 1
#define ALPA_EXEC_EAGER 0
#define ALPA_EXEC_GRAPH 1
/* Topology (pipeline.hpp:48). */
#define ALPA_TOPOLOGY_MULTI 0
#define ALPA_TOPOLOGY_SINGLE 1

typedef struct alpa_ctx alpa_ctx;

/* ModelConfig (model.hpp:12-29).  vision_blocks, hidden_dim, vocab_size and
 * patch_size only position the action weights inside the reference's single
 * splitmix64 weight stream (model.cpp:120-151). */
typedef struct alpa_model_cfg {
    int64_t vision_blocks;
    int64_t decoder_blocks;
    int64_t hidden_dim;
    int64_t action_hidden_dim;
    int64_t kv_dim;
    int64_t heads;
    int64_t vocab_size;
    int64_t patch_size;
    int64_t action_steps;    /* must be 64 (model.cpp:20) */
    int64_t diffusion_iters; /* K */
    float update_scale;      /* Euler step, default 0.1 (model.hpp:23) */
    int32_t dtype;           /* ALPA_DTYPE_* */
    uint64_t weight_seed;
} alpa_model_cfg;

/* InferenceRequest fields the path consumes (pipeline.hpp:97-113). */
typedef struct alpa_request {
    int64_t num_trajectories;    /* N lanes on this context                     */
    int64_t lane0;               /* global index of lane 0 (multi-GPU slices keep
                                    global noise seeds)         */
    uint64_t action_init_seed;   /* lane l seed = seed + (lane0+l)*stride        */
    uint64_t action_seed_stride;
    int64_t diffusion_iters;     /* K; <= 0 -> cfg.diffusion_iters              */
    int32_t topology;            /* ALPA_TOPOLOGY_*                             */
    int32_t kv_strategy;         /* ALPA_KV_* (accepted; layout is always static)*/
    int32_t executor;            /* ALPA_EXEC_*                                 */
    float v0;                    /* initial speed (initial_speed_from_history)  */
} alpa_request;

/* Per-call counters (redefined from DispatchStats, substrate.hpp:68-73). */
typedef struct alpa_stats {
    double device_ms;            /* CUDA-event time of the refine+rollout        */
    int64_t kernel_launches;     /* kernels executed by the device timeline      */
    int64_t graph_launches;      /* 1 when the K loop replayed as one graph      */
    int64_t graph_nodes;         /* kernel nodes in the captured graph           */
    int64_t kv_bytes;            /* footprint_bytes() equivalent (kv_cache.cpp:365)*/
    int64_t h2d_bytes;
    int64_t d2h_bytes;
    /* per diffusion iteration device time (LatencyReport::action_gen_iter_ms,
     * profiler.hpp:36): events between the iterations, inside the graph too */
    int64_t n_iter;              /* iterations recorded (<= ALPA_MAX_ITER_MS)    */
    double iter_ms[64];
    int64_t bytes_allocated;     /* device bytes owned by the context            */
} alpa_stats;
#define ALPA_MAX_ITER_MS 64

/* ---- context ------------------------------------------------------------ */
int alpa_ctx_create(const alpa_model_cfg* cfg, int device, alpa_ctx** out);
void alpa_ctx_destroy(alpa_ctx* ctx);
/* Message of the last failing call on ctx (ctx may be NULL: thread-local). */
const char* alpa_last_error(const alpa_ctx* ctx);
/* Run on a caller stream (cudaStream_t as void*); NULL = ctx-owned stream. */
int alpa_set_stream(alpa_ctx* ctx, void* cuda_stream);
/* Default cfg (fixtures/default_config.json model block). */
void alpa_default_cfg(alpa_model_cfg* cfg);
int alpa_validate_cfg(const alpa_model_cfg* cfg); /* ModelConfig::validate, model.cpp:9-24 */

/* ---- weights ------------------------------------------------------------ */
/* Draws the action expert on device from the splitmix64 stream of weight_seed,
 * jumping stream_offset draws (<0: offset implied by cfg, model.cpp:120-140). */
int alpa_load_weights_seeded(alpa_ctx* ctx, uint64_t weight_seed, int64_t stream_offset);
/* Host arena in ModelWeights draw order (action_in, mlp1, mlp2, blocks(q,k,v,o,
 * mlp1,mlp2; w [in][out] then b), head); count = alpa_action_param_count(). */
int alpa_load_weights_host(alpa_ctx* ctx, const float* arena, int64_t count);
int64_t alpa_weight_stream_offset(const alpa_model_cfg* cfg);
int64_t alpa_action_param_count(const alpa_model_cfg* cfg);

/* ---- prefix (the sealed reasoning KV; one copy, read-only) ------------ */
/* Host f32 [n_prefix][B][2][r][kv]; n_prefix = 1 for single topology. */
int alpa_bind_prefix(alpa_ctx* ctx, const float* kv, int64_t n_prefix, int64_t r);
/* Device buffer in the context dtype layout (f32 or bf16), same shape; the
 * context keeps the pointer (e.g. after an NCCL broadcast into it). */
int alpa_bind_prefix_device(alpa_ctx* ctx, const void* kv, int64_t n_prefix, int64_t r);
/* make_sealed_cache recipe (tests/test_model.cpp:43-74) generated on device:
 * per block Rng(seed+b) uniform(-0.5,0.5) keys, V = -K. */
int alpa_bind_prefix_synthetic(alpa_ctx* ctx, uint64_t seed, int64_t r);
/* Writes the make_sealed_cache recipe for `seed` into a caller device buffer
 * [B][2][r][kv] in the ctx dtype (scene producer for benches / collectives);
 * bind it with alpa_bind_prefix_device. */
int alpa_synthesize_prefix(alpa_ctx* ctx, void* dst, uint64_t seed, int64_t r);
/* Device pointer/bytes of the bound prefix (for collectives). */
int alpa_prefix_device(alpa_ctx* ctx, void** ptr, int64_t* bytes);
/* Multi topology: lane l attends prefix lane_map[l] (default: all 0). */
int alpa_set_lane_prefix(alpa_ctx* ctx, const int32_t* lane_map, int64_t n);

/* ---- reasoning-stage KV producer --------------------------
 * The language model's prefill / decode on the device, writing every token's
 * K/V in place into a static-capacity buffer in the action stage's prefix
 * layout [lanes][B][2][capacity][kv] (context dtype); seal binds it as the
 * prefix with no copy.  The caller keeps the vision encoder, the tokenizer and
 * the sampler loop, like Engine::reasoning_pass (pipeline.cpp:247-390). */
/* KvCache(static) with reasoning_capacity = T + max_new_tokens
 * (pipeline.cpp:281-288); lanes = 1 (single topology) or N (multi). Unbinds a
 * prefix the context produced earlier. */
int alpa_reasoning_begin(alpa_ctx* ctx, int64_t lanes, int64_t capacity);
/* Model::prefill (model.cpp:408-464) over ctx = [vision rows | prompt
 * embeddings] + positions (pipeline.cpp:297-325): vision_rows [lanes][P][hidden]
 * host f32 (may be NULL when P == 0), prompt_ids [n_prompt]; then
 * logits_head (model.cpp:509-513): logits_out [lanes][vocab] host. */
int alpa_reasoning_prefill(alpa_ctx* ctx, const float* vision_rows, int64_t P,
                           const int64_t* prompt_ids, int64_t n_prompt, float* logits_out);
/* One decode step (pipeline.cpp:368-386, Model::decode_step model.cpp:484-507):
 * token_ids [lanes] at the next position, K/V appended, logits_out [lanes][vocab]. */
int alpa_reasoning_decode(alpa_ctx* ctx, const int64_t* token_ids, float* logits_out);
/* KvCache::seal_reasoning (kv_cache.cpp:181-190): bind the produced KV as the
 * action stage's prefix (n_prefix = lanes, r = tokens appended, in place). */
int alpa_reasoning_seal(alpa_ctx* ctx, int64_t* r_out);
/* sample_token (model.cpp:30-54) on the host, bit-exact: greedy argmax, or
 * the temperature-1 softmax CDF walk in double with the Rng state (splitmix64,
 * common.hpp:36-59) advanced in place; InternalError on NaN logits. */
int alpa_sample_token(const float* logits, int64_t vocab, int stochastic, uint64_t* rng_state,
                      int64_t* token_out);

/* ---- the path ----------------------------------------------------------- */
/* Host in, host out: host noise (bit-exact Rng::normal) -> H2D -> K-step
 * refine (one CUDA graph) -> device rollout -> D2H.  actions_out [N][64][2],
 * traj_out [N][64][3] (either may be NULL). */
int alpa_generate(alpa_ctx* ctx, const alpa_request* req, float* actions_out,
                  float* traj_out, alpa_stats* stats);
/* Device-resident variant: d_noise [N][64][2] already in HBM; results stay in
 * HBM (d_actions [N][64][2], d_traj [N][64][3]; d_traj may be NULL). */
int alpa_generate_device(alpa_ctx* ctx, const alpa_request* req, const float* d_noise,
                         float* d_actions, float* d_traj, alpa_stats* stats);
/* The rollout's non-finite-action flag of the last generate call (device int,
 * non-zero = InternalError "non-finite action", pipeline.cpp:133-135).
 * alpa_generate checks it itself; alpa_generate_device checks it when `stats`
 * is given (the call synchronises then) and otherwise leaves it to the caller,
 * who reads it after synchronising the context's stream. */
int alpa_last_rollout_flag_device(alpa_ctx* ctx, const int** flag);

/* ---- measurement --------------------------------------------------------- */
/* Per-kernel device time of `iters` eagerly launched iterations (+ rollout),
 * an event pair around every launch, aggregated by kernel name; flops/bytes
 * are the algorithmic work of those launches (SURVEY.md §8d accounting). */
typedef struct alpa_kernel_prof {
    char name[40];
    int64_t launches;
    double total_ms;
    double flops;
    double bytes;
} alpa_kernel_prof;
int alpa_profile(alpa_ctx* ctx, const alpa_request* req, int64_t iters, alpa_kernel_prof* out,
                 int32_t max_out, int32_t* n_out);
/* Diagnostics: per-CTA event times [n_ops][grid][16] (globaltimer ns) of the
 * last profiled persistent-kernel iteration; needs ALPA_MK_TRACE=1 in the
 * environment when the plan was built.  Events: 0 inputs ready (producer),
 * 1 first stage landed (MMA), 2 last MMA issued, 3 accumulator ready
 * (epilogue), 4 split rendezvous, 5 item published, 6 weight stages issued,
 * 7 accumulator drained, 8 fixup done, 9 publish fences passed. */
int alpa_debug_mk_trace(alpa_ctx* ctx, unsigned long long* out, int64_t max_elems,
                        int64_t* n_ops, int64_t* grid);

/* ---- open-loop evaluation (eval.cpp:14-59), bit-exact fp64 -------------- */
/* Batch of scenes: traj [scenes][n][steps][3] (x, y, yaw), gt [scenes][steps][3];
 * outputs min_ade [scenes] (minivla::min_ade) and diversity [scenes]
 * (minivla::diversity); either output may be NULL.  Errors like the reference:
 * n < 1 -> ALPA_ERR_INTERNAL ("min_ade: no samples"), diversity with n < 2 ->
 * ALPA_ERR_INTERNAL.  Host-buffer variant and device-pointer variant. */
int alpa_eval_open_loop(alpa_ctx* ctx, const float* traj, const float* gt, int64_t scenes, int64_t n,
                        int64_t steps, double* min_ade, double* diversity);
int alpa_eval_open_loop_device(alpa_ctx* ctx, const float* d_traj, const float* d_gt, int64_t scenes,
                               int64_t n, int64_t steps, double* d_min_ade, double* d_diversity);

/* ---- host helpers (bit-exact restatements of the reference host code) -- */
/* Rng::normal noise for lanes [lane0, lane0+n): out [n][steps][2]. */
void alpa_host_noise(uint64_t seed, uint64_t stride, int64_t lane0, int64_t n,
                     int64_t steps, float* out);
/* initial_speed_from_history (pipeline.cpp:150-156): history [16][3]. */
float alpa_initial_speed(const float* history);
/* Device rollout of host actions [n][64][2] -> traj [n][64][3]. */
int alpa_rollout(alpa_ctx* ctx, const float* actions, int64_t n, float v0, float* traj);
int64_t alpa_kv_footprint_bytes(int64_t blocks, int64_t batch, int64_t tokens,
                                int64_t kv_dim, int64_t elem_bytes);
/* Build/ABI identification string. */
const char* alpa_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ALPA_ACTION_H */
