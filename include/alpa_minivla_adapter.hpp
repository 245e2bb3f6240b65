// Drop-in adapter for the reference's own types: routes
// minivla::Engine::run_action_generation (pipeline.cpp:399-436) to the B200
// library (alpa_action.h) WITHOUT any mirror types.  Compile it inside the
// reference's build (it includes <minivla/pipeline.hpp>); INTEGRATION.md shows
// the two-line change in Engine::infer that calls it.
//
//   minivla::Engine engine(cfg);
//   alpa_minivla::ActionStage gpu(cfg);                  // weights drawn on device
//   minivla::ReasoningOutput r = engine.run_reasoning(req);
//   std::vector<minivla::ActionSequence> a =
//       gpu.run_action_generation(engine.substrate(), r, req);   // was engine.run_action_generation(r, req)
//
// What it reads: the sealed reasoning KvCache of `reasoning`, one substrate
// buffer per block shaped [2(K,V)][batch][cap][kv_dim] f32 (kv_cache.cpp:11-14,
// region offset ((s*batch + lane)*cap + t)*kv), through Substrate::read
// (substrate.hpp:128).  The first reasoning_len(b) tokens of every block and
// lane are packed to the library's [batch][B][2][r][kv] layout and bound once
// per call (alpa_bind_prefix): the reference uses the KV it is handed on every
// call, so does this adapter.  Single topology with N > 1 does NOT replicate
// the cache (replicate_for_batch, kv_cache.cpp:280-318, is what the library
// removes): every lane attends the one prefix in place.
//
// Error behaviour (the reference's exception types, common.hpp:12-23):
//   unsealed cache                      -> InternalError (kv_cache.cpp:195)
//   kv batch != N (N < 1 included)      -> InternalError (pipeline.cpp:411-413)
//   single topology, cache batch != 1   -> InternalError (kv_cache.cpp:281-283)
//   graph executor + dynamic kv         -> ConfigError   (model.cpp:609-611)
//   anything else the library reports   -> mapped by its return code (1/2/3)
#pragma once

#include <minivla/common.hpp>
#include <minivla/kv_cache.hpp>
#include <minivla/model.hpp>
#include <minivla/pipeline.hpp>
#include <minivla/substrate.hpp>

#include <cstdint>
#include <string>
#include <vector>

#include "alpa_action.h"

namespace alpa_minivla {

inline void check(int rc, alpa_ctx* ctx) {
    if (rc == ALPA_OK) return;
    const std::string msg = ctx ? alpa_last_error(ctx) : "alpa: context creation failed";
    if (rc == ALPA_ERR_IO) throw minivla::IoError(msg);
    if (rc == ALPA_ERR_CONFIG) throw minivla::ConfigError(msg);
    throw minivla::InternalError(msg);
}

inline alpa_model_cfg to_c(const minivla::ModelConfig& m, int dtype) {
    alpa_model_cfg c{};
    alpa_default_cfg(&c);
    c.vision_blocks = m.vision_blocks;
    c.decoder_blocks = m.decoder_blocks;
    c.hidden_dim = m.hidden_dim;
    c.action_hidden_dim = m.action_hidden_dim;
    c.kv_dim = m.kv_dim;
    c.heads = m.heads;
    c.vocab_size = m.vocab_size;
    c.patch_size = m.patch_size;
    c.action_steps = m.action_steps;
    c.diffusion_iters = m.diffusion_iters;
    c.update_scale = m.update_scale;
    c.dtype = dtype;
    c.weight_seed = m.weight_seed;
    return c;
}

class ActionStage {
public:
    // dtype ALPA_DTYPE_F32: the reference's arithmetic (rel-L2 <= 1e-4);
    // ALPA_DTYPE_BF16: the tensor-core path (rel-L2 <= 2e-2).
    explicit ActionStage(const minivla::ModelConfig& cfg, int device = 0, int dtype = ALPA_DTYPE_F32)
        : cfg_(cfg) {
        cfg.validate();  // model.cpp:9-24 (throws ConfigError)
        const alpa_model_cfg c = to_c(cfg, dtype);
        check(alpa_ctx_create(&c, device, &ctx_), ctx_);
        // ModelWeights::build's stream (model.cpp:120-151): the same seed, the
        // action expert's draws found by jump-ahead
        check(alpa_load_weights_seeded(ctx_, cfg.weight_seed, -1), ctx_);
    }
    ~ActionStage() { alpa_ctx_destroy(ctx_); }
    ActionStage(const ActionStage&) = delete;
    ActionStage& operator=(const ActionStage&) = delete;

    alpa_ctx* handle() { return ctx_; }

    // Engine::run_action_generation (pipeline.hpp:145-148), same arguments plus
    // the substrate that owns the reasoning cache (Engine::substrate()).
    std::vector<minivla::ActionSequence> run_action_generation(const minivla::Substrate& sub,
                                                               minivla::ReasoningOutput& reasoning,
                                                               const minivla::InferenceRequest& request,
                                                               minivla::Model::DiffusionResult* diff = nullptr,
                                                               std::int64_t* kv_bytes = nullptr) {
        const std::int64_t n = request.num_trajectories;
        const minivla::KvCache& kv = reasoning.kv;
        if (!kv.sealed()) throw minivla::InternalError("kv cache: action KV write before reasoning sealed");
        const std::int64_t batch = kv.layout().batch;
        if (request.topology == minivla::Topology::Single && n > 1 && batch != 1)
            throw minivla::InternalError("replicate_for_batch: source cache must have batch 1");
        const std::int64_t eff = (request.topology == minivla::Topology::Single && n > 1) ? n : batch;
        if (eff != n) throw minivla::InternalError("kv batch does not match the requested trajectory count");
        bind(sub, kv);
        std::vector<minivla::ActionSequence> out = generate(request, diff, kv_bytes);
        return out;
    }

private:
    std::vector<minivla::ActionSequence> generate(const minivla::InferenceRequest& request,
                                                  minivla::Model::DiffusionResult* diff = nullptr,
                                                  std::int64_t* kv_bytes = nullptr) {
        const std::int64_t n = request.num_trajectories;
        alpa_request r{};
        r.num_trajectories = n;
        r.lane0 = 0;
        r.action_init_seed = request.action_init_seed;
        r.action_seed_stride = request.action_seed_stride;
        r.diffusion_iters = 0;  // ModelConfig::diffusion_iters
        r.topology = request.topology == minivla::Topology::Single ? ALPA_TOPOLOGY_SINGLE : ALPA_TOPOLOGY_MULTI;
        r.kv_strategy = request.kv_strategy == minivla::KvStrategy::Static ? ALPA_KV_STATIC : ALPA_KV_DYNAMIC;
        r.executor = request.executor == minivla::ExecMode::Graph ? ALPA_EXEC_GRAPH : ALPA_EXEC_EAGER;
        r.v0 = minivla::initial_speed_from_history(request.pose_history);
        const std::int64_t A = cfg_.action_steps;
        std::vector<float> acts(static_cast<size_t>(n * A * 2));
        alpa_stats st{};
        // actions only: trajectory validation stays in postprocessing, as in the reference
        check(alpa_generate(ctx_, &r, acts.data(), nullptr, &st), ctx_);
        std::vector<minivla::ActionSequence> out(static_cast<size_t>(n));
        for (std::int64_t l = 0; l < n; ++l) {  // Model::read_actions (model.cpp:638-650)
            out[l].steps.resize(static_cast<size_t>(A));
            for (std::int64_t i = 0; i < A; ++i)
                out[l].steps[i] = minivla::ActionStep{acts[(l * A + i) * 2], acts[(l * A + i) * 2 + 1]};
        }
        if (kv_bytes) *kv_bytes = st.kv_bytes;
        if (diff) {
            diff->actions = out;
            diff->iter_ms.assign(st.iter_ms, st.iter_ms + st.n_iter);
            // substrate dispatch deltas do not exist on this path (one graph launch)
            diff->iter_stats.assign(static_cast<size_t>(st.n_iter), minivla::DispatchStats{});
            diff->graph_commands = st.graph_nodes;
        }
        last_ = st;
        return out;
    }

public:
    // actions_to_trajectory (pipeline.cpp:124-148) on the device, bit-exact
    // with the reference's fp64 host loop; throws InternalError like it.
    minivla::Trajectory actions_to_trajectory(const minivla::ActionSequence& a, float initial_speed) {
        const std::int64_t A = static_cast<std::int64_t>(a.steps.size());
        std::vector<float> in(static_cast<size_t>(A * 2)), o(static_cast<size_t>(A * 3));
        for (std::int64_t i = 0; i < A; ++i) {
            in[i * 2] = a.steps[i].accel;
            in[i * 2 + 1] = a.steps[i].curvature;
        }
        check(alpa_rollout(ctx_, in.data(), 1, initial_speed, o.data()), ctx_);
        minivla::Trajectory t;
        t.poses.resize(static_cast<size_t>(A));
        for (std::int64_t i = 0; i < A; ++i) t.poses[i] = minivla::Pose{o[i * 3], o[i * 3 + 1], o[i * 3 + 2]};
        return t;
    }

    const alpa_stats& last_stats() const { return last_; }

    // Engine::run_reasoning with the KV produced ON THE DEVICE:
    // the reference engine keeps the vision encoder and the tokenizer
    // (Engine::preprocess, Model::vision_encode on the lane-tiled patch rows,
    // pipeline.cpp:265-277); the language model's prefill / decode run in the
    // library and append K/V in place into the action stage's layout
    // (static capacity T + max_new_tokens, pipeline.cpp:281-286); the decode
    // loop is reasoning_pass's (pipeline.cpp:330-388) with the reference's
    // sampler (alpa_sample_token, bit-exact).  The sealed KV stays bound in the
    // library: run_action_generation_device() then attends it with no copy.
    struct DeviceReasoning {
        std::vector<std::vector<std::int64_t>> cot_tokens;  // per lane, no terminator
        std::int64_t token_count = 0;                       // decode steps executed
        std::int64_t prompt_tokens = 0;                     // T
        std::int64_t reasoning_len = 0;                     // r = T + token_count
    };
    DeviceReasoning run_reasoning(minivla::Engine& engine, const minivla::InferenceRequest& request) {
        minivla::Engine::validate_request(request);
        const minivla::ModelConfig& m = engine.config();
        const std::int64_t lanes = request.topology == minivla::Topology::Multi ? request.num_trajectories : 1;
        const minivla::Engine::Preprocessed pre = engine.preprocess(request);
        minivla::Substrate& sub = engine.substrate();
        const std::int64_t P = pre.patches, h = m.hidden_dim, V = m.vocab_size;
        std::vector<float> tiled(static_cast<size_t>(lanes * P * pre.patch_dim));
        for (std::int64_t l = 0; l < lanes; ++l)
            std::copy(pre.patch_rows.begin(), pre.patch_rows.end(), tiled.begin() + l * P * pre.patch_dim);
        const std::size_t mark = sub.alloc_mark();
        const minivla::BufferId patch = sub.alloc({lanes * P, pre.patch_dim});
        sub.write(patch, tiled);
        const minivla::BufferId vis = engine.model().vision_encode(patch, lanes, P);
        const auto vrows = sub.read(vis);
        std::vector<float> vision(vrows.begin(), vrows.end());  // [lanes][P][h]
        sub.free_allocated_since(mark);
        const std::vector<std::int64_t>& prompt = pre.prompt.ids;
        const std::int64_t T = P + static_cast<std::int64_t>(prompt.size());
        check(alpa_reasoning_begin(ctx_, lanes, T + m.max_new_tokens), ctx_);
        std::vector<float> logits(static_cast<size_t>(lanes * V));
        check(alpa_reasoning_prefill(ctx_, vision.data(), P, prompt.data(), static_cast<std::int64_t>(prompt.size()),
                                     logits.data()),
              ctx_);
        DeviceReasoning out;
        out.cot_tokens.assign(static_cast<size_t>(lanes), {});
        out.prompt_tokens = T;
        std::vector<std::uint64_t> rng(static_cast<size_t>(lanes));
        for (std::int64_t l = 0; l < lanes; ++l) rng[l] = request.sampler_seed + static_cast<std::uint64_t>(l);
        std::vector<bool> done(static_cast<size_t>(lanes), false);
        const bool forced = request.forced_cot_tokens > 0;
        const std::int64_t max_m = forced ? std::min(request.forced_cot_tokens, m.max_new_tokens) : m.max_new_tokens;
        const int stochastic = request.sampler_mode == minivla::SampleMode::Stochastic ? 1 : 0;
        const std::int64_t term = engine.tokenizer().termination_token();
        std::vector<std::int64_t> ids(static_cast<size_t>(lanes));
        std::int64_t steps = 0;
        while (steps < max_m) {
            bool all_done = true;
            for (std::int64_t l = 0; l < lanes; ++l) all_done = all_done && done[l];
            if (all_done && !forced) break;
            for (std::int64_t l = 0; l < lanes; ++l) {
                check(alpa_sample_token(logits.data() + l * V, V, stochastic, &rng[l], &ids[l]), nullptr);
                if (!done[l]) {
                    if (!forced && ids[l] == term) done[l] = true;
                    else out.cot_tokens[l].push_back(ids[l]);
                }
            }
            steps += 1;
            check(alpa_reasoning_decode(ctx_, ids.data(), logits.data()), ctx_);
        }
        out.token_count = steps;
        check(alpa_reasoning_seal(ctx_, &out.reasoning_len), ctx_);
        (void)h;
        return out;
    }

    // Engine::run_action_generation on the KV run_reasoning left on the device.
    std::vector<minivla::ActionSequence> run_action_generation_device(const minivla::InferenceRequest& request) {
        return generate(request);
    }

private:
    // Pack the sealed reasoning tokens of every block / lane into
    // [batch][B][2][r][kv] f32 and bind them (the library converts to its dtype).
    void bind(const minivla::Substrate& sub, const minivla::KvCache& kv) {
        const std::int64_t B = kv.layout().num_blocks, batch = kv.layout().batch, kd = kv.layout().kv_dim;
        const std::int64_t r = kv.reasoning_len(0);
        for (std::int64_t b = 1; b < B; ++b)
            if (kv.reasoning_len(b) != r) throw minivla::InternalError("kv cache: ragged reasoning lengths");
        packed_.assign(static_cast<size_t>(batch * B * 2 * r * kd), 0.0f);
        for (std::int64_t b = 0; b < B; ++b) {
            const auto span = sub.read(kv.block_buffer(b));
            const std::int64_t cap = static_cast<std::int64_t>(span.size()) / (2 * batch * kd);
            if (cap < r) throw minivla::InternalError("kv cache: block buffer smaller than the reasoning length");
            for (std::int64_t s = 0; s < 2; ++s)
                for (std::int64_t l = 0; l < batch; ++l) {
                    const float* src = span.data() + ((s * batch + l) * cap) * kd;  // region_offset, t = 0
                    float* dst = packed_.data() + (((l * B + b) * 2 + s) * r) * kd;
                    std::copy(src, src + r * kd, dst);
                }
        }
        check(alpa_bind_prefix(ctx_, packed_.data(), batch, r), ctx_);
    }

    minivla::ModelConfig cfg_;
    alpa_ctx* ctx_ = nullptr;
    std::vector<float> packed_;
    alpa_stats last_{};
};

}  // namespace alpa_minivla
