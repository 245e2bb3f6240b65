// alpa_minivla_shim.hpp -- header-only C++ re-exposure of the reference's
// action-generation API (minivla, /root/reference/proj) over the C-ABI in
// alpa_action.h.  A reference caller swaps
//
//     minivla::Engine::run_action_generation      pipeline.hpp:145-148
//     minivla::actions_to_trajectory              pipeline.hpp:90
//     minivla::initial_speed_from_history         pipeline.hpp:93
//
// for the same-named members below; argument meaning and the exception types
// (ConfigError / IoError / InternalError, common.hpp:12-23) are unchanged.
// The reasoning stage is out of scope: ReasoningOutput carries the sealed
// prefix KV as a host f32 buffer [n_prefix][B][2][r][kv] (what
// Substrate::read(kv.block_buffer(b)) yields, first r tokens per block) or a
// device pointer in the context dtype.
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <atomic>
#include <cstdio>
#include <string>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "alpa_action.h"

namespace alpa_shim {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : Error {
    using Error::Error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct InternalError : Error {
    using Error::Error;
};

inline void check(int rc, const alpa_ctx* ctx) {
    if (rc == ALPA_OK) return;
    const std::string msg = alpa_last_error(ctx);
    if (rc == ALPA_ERR_IO) throw IoError(msg);
    if (rc == ALPA_ERR_CONFIG) throw ConfigError(msg);
    throw InternalError(msg);
}

enum class Topology { Multi, Single };           // pipeline.hpp:48
enum class KvStrategy { Dynamic, Static };       // kv_cache.hpp:9
enum class ExecMode { Eager, Graph };            // model.hpp:43
enum class Dtype { F32 = ALPA_DTYPE_F32, BF16 = ALPA_DTYPE_BF16 };

// ModelConfig (model.hpp:12-29) + compute dtype.
struct ModelConfig {
    std::int64_t vision_blocks = 4;
    std::int64_t decoder_blocks = 6;
    std::int64_t hidden_dim = 64;
    std::int64_t action_hidden_dim = 32;
    std::int64_t kv_dim = 32;
    std::int64_t heads = 4;
    std::int64_t vocab_size = 512;
    std::int64_t patch_size = 14;
    std::int64_t action_steps = 64;
    std::int64_t diffusion_iters = 10;
    float update_scale = 0.1f;
    std::int64_t max_new_tokens = 256;
    std::uint64_t weight_seed = 1234;
    Dtype dtype = Dtype::F32;

    alpa_model_cfg c() const {
        alpa_model_cfg m{};
        m.vision_blocks = vision_blocks;
        m.decoder_blocks = decoder_blocks;
        m.hidden_dim = hidden_dim;
        m.action_hidden_dim = action_hidden_dim;
        m.kv_dim = kv_dim;
        m.heads = heads;
        m.vocab_size = vocab_size;
        m.patch_size = patch_size;
        m.action_steps = action_steps;
        m.diffusion_iters = diffusion_iters;
        m.update_scale = update_scale;
        m.dtype = static_cast<int32_t>(dtype);
        m.weight_seed = weight_seed;
        return m;
    }
    void validate() const {  // ModelConfig::validate, model.cpp:9-24
        const alpa_model_cfg m = c();
        check(alpa_validate_cfg(&m), nullptr);
    }
};

struct ActionStep {  // model.hpp:31-34
    float accel = 0.0f;
    float curvature = 0.0f;
};
struct ActionSequence {  // model.hpp:38-40
    std::vector<ActionStep> steps;
};
struct Pose {  // pipeline.hpp:18-22
    float x = 0.0f, y = 0.0f, yaw = 0.0f;
};
struct PoseHistory {
    std::array<Pose, 16> poses{};
};
struct Trajectory {
    std::vector<Pose> poses;
};

// The InferenceRequest fields the path consumes (pipeline.hpp:97-113).
enum class SampleMode { Greedy, Stochastic };

struct InferenceRequest {
    PoseHistory pose_history;
    std::int64_t num_trajectories = 1;
    Topology topology = Topology::Multi;
    KvStrategy kv_strategy = KvStrategy::Dynamic;
    ExecMode executor = ExecMode::Eager;
    std::uint64_t action_init_seed = 2;
    std::uint64_t action_seed_stride = 1;
    // reasoning stage (pipeline.hpp:95-111)
    std::uint64_t sampler_seed = 1;
    SampleMode sampler_mode = SampleMode::Stochastic;
    std::int64_t forced_cot_tokens = 0;
};

// Sealed reasoning prefix (the part of ReasoningOutput the path reads,
// pipeline.hpp:120-126).
struct ReasoningOutput {
    std::vector<float> kv_host;   // [n_prefix][B][2][r][kv] f32, or empty
    const void* kv_device = nullptr;  // same shape, context dtype, or null
    std::int64_t n_prefix = 1;
    std::int64_t reasoning_len = 0;   // r
    // Identity of the content, advanced by the shim itself: every new object
    // gets a fresh id; callers that edit kv_host / the device buffer IN PLACE
    // call touch().  run_action_generation rebinds whenever (id, version, data
    // pointers, shape) differ from the last bind.
    std::uint64_t id = next_id();
    std::uint64_t version = 0;
    void touch() { ++version; }
    // produced by Engine::run_reasoning_device: the KV already sits bound inside
    // the library (static capacity, in place) -- nothing to upload
    bool device_resident = false;
    std::vector<std::vector<std::int64_t>> cot_tokens;  // per lane, no terminator
    std::int64_t token_count = 0;                       // decode steps executed
    std::int64_t prompt_tokens = 0;                     // T

private:
    static std::uint64_t next_id() {
        static std::atomic<std::uint64_t> ctr{1};
        return ctr.fetch_add(1);
    }
};

// Model::DiffusionResult (model.hpp:155-160), counters redefined: one graph
// launch per call, kernel nodes instead of substrate commands.
struct DiffusionResult {
    std::vector<double> iter_ms;
    std::int64_t graph_commands = 0;
    std::int64_t graph_launches = 0;
    double device_ms = 0.0;
};

// minivla::LatencyReport (profiler.hpp:31-46) and its JSON wire format
// (profiler.cpp:31-46: same keys, numbers printed round-trip exact).
struct LatencyReport {
    std::array<double, 5> component_ms{};  // preprocessing, reasoning vision/prefill/decode, action gen
    double total_ms = 0.0;
    double postprocessing_ms = 0.0;
    int repeats = 1;
    std::vector<double> action_gen_iter_ms;
    std::uint64_t alloc_count = 0;
    std::uint64_t dispatch_count = 0;
    std::uint64_t replay_count = 0;
    std::uint64_t bytes_allocated = 0;
    std::int64_t kv_bytes = 0;
    std::int64_t cot_tokens = 0;

    std::string to_json() const {
        static const char* keys[5] = {"preprocessing_ms", "reasoning_vision_ms", "reasoning_prefill_ms",
                                      "reasoning_decode_ms", "action_gen_ms"};
        auto num = [](double v) {
            char b[40];
            std::snprintf(b, sizeof b, "%.17g", v);
            return std::string(b);
        };
        std::string j = "{";
        for (int i = 0; i < 5; ++i) j += "\"" + std::string(keys[i]) + "\":" + num(component_ms[i]) + ",";
        j += "\"total_ms\":" + num(total_ms) + ",\"postprocessing_ms\":" + num(postprocessing_ms) +
             ",\"repeats\":" + std::to_string(repeats) + ",\"action_gen_iter_ms\":[";
        for (size_t i = 0; i < action_gen_iter_ms.size(); ++i)
            j += (i ? "," : "") + num(action_gen_iter_ms[i]);
        j += "],\"alloc_count\":" + std::to_string(alloc_count) + ",\"dispatch_count\":" +
             std::to_string(dispatch_count) + ",\"replay_count\":" + std::to_string(replay_count) +
             ",\"bytes_allocated\":" + std::to_string(bytes_allocated) + ",\"kv_bytes\":" +
             std::to_string(kv_bytes) + ",\"cot_tokens\":" + std::to_string(cot_tokens) + "}";
        return j;
    }
};

inline float initial_speed_from_history(const PoseHistory& h) {  // pipeline.cpp:150-156
    float buf[16 * 3];
    for (int i = 0; i < 16; ++i) {
        buf[i * 3] = h.poses[i].x;
        buf[i * 3 + 1] = h.poses[i].y;
        buf[i * 3 + 2] = h.poses[i].yaw;
    }
    return alpa_initial_speed(buf);
}

// The action-generation half of minivla::Engine on one GPU context.
class Engine {
public:
    explicit Engine(const ModelConfig& cfg, int device = 0) : cfg_(cfg) {
        const alpa_model_cfg m = cfg.c();
        check(alpa_ctx_create(&m, device, &ctx_), nullptr);
        check(alpa_load_weights_seeded(ctx_, cfg.weight_seed, -1), ctx_);
    }
    ~Engine() { alpa_ctx_destroy(ctx_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    const ModelConfig& config() const { return cfg_; }
    alpa_ctx* handle() { return ctx_; }

    // Engine::run_action_generation (pipeline.cpp:399-436): no prefix
    // replication (every lane attends the single prefix copy in place).
    std::vector<ActionSequence> run_action_generation(ReasoningOutput& reasoning,
                                                      const InferenceRequest& request,
                                                      DiffusionResult* diff = nullptr,
                                                      std::int64_t* kv_bytes = nullptr) {
        bind(reasoning);
        const std::int64_t n = request.num_trajectories;
        const std::int64_t A = cfg_.action_steps;
        alpa_request r = to_c(request);
        std::vector<float> acts(static_cast<size_t>(n > 0 ? n : 0) * A * 2);
        alpa_stats st{};
        check(alpa_generate(ctx_, &r, acts.data(), nullptr, &st), ctx_);
        if (kv_bytes) *kv_bytes = st.kv_bytes;
        last_stats_ = st;
        if (diff) {
            // per-iteration device times (timing events between the iterations)
            diff->iter_ms.assign(st.iter_ms, st.iter_ms + st.n_iter);
            diff->graph_commands = st.graph_nodes;
            diff->graph_launches = st.graph_launches;
            diff->device_ms = st.device_ms;
        }
        std::vector<ActionSequence> out(static_cast<size_t>(n));
        for (std::int64_t l = 0; l < n; ++l) {
            out[l].steps.resize(static_cast<size_t>(A));
            for (std::int64_t i = 0; i < A; ++i)
                out[l].steps[i] = {acts[(l * A + i) * 2], acts[(l * A + i) * 2 + 1]};
        }
        return out;
    }

    // run_action_generation + the postprocessing rollout in one device pass
    // (Engine::infer's action-gen + postprocessing, pipeline.cpp:462-479).
    std::vector<Trajectory> generate_trajectories(ReasoningOutput& reasoning,
                                                  const InferenceRequest& request,
                                                  std::vector<ActionSequence>* actions = nullptr) {
        bind(reasoning);
        const std::int64_t n = request.num_trajectories;
        const std::int64_t A = cfg_.action_steps;
        alpa_request r = to_c(request);
        std::vector<float> acts(static_cast<size_t>(n > 0 ? n : 0) * A * 2);
        std::vector<float> traj(static_cast<size_t>(n > 0 ? n : 0) * A * 3);
        check(alpa_generate(ctx_, &r, acts.data(), traj.data(), nullptr), ctx_);
        std::vector<Trajectory> out(static_cast<size_t>(n));
        if (actions) actions->assign(static_cast<size_t>(n), ActionSequence{});
        for (std::int64_t l = 0; l < n; ++l) {
            out[l].poses.resize(static_cast<size_t>(A));
            for (std::int64_t i = 0; i < A; ++i) {
                const float* p = &traj[(l * A + i) * 3];
                out[l].poses[i] = {p[0], p[1], p[2]};
            }
            if (actions) {
                (*actions)[l].steps.resize(static_cast<size_t>(A));
                for (std::int64_t i = 0; i < A; ++i)
                    (*actions)[l].steps[i] = {acts[(l * A + i) * 2], acts[(l * A + i) * 2 + 1]};
            }
        }
        return out;
    }

    // actions_to_trajectory (pipeline.cpp:124-148) on the device, bit-exact.
    Trajectory actions_to_trajectory(const ActionSequence& a, float initial_speed) {
        const std::int64_t A = static_cast<std::int64_t>(a.steps.size());
        std::vector<float> in(static_cast<size_t>(A) * 2), out(static_cast<size_t>(A) * 3);
        for (std::int64_t i = 0; i < A; ++i) {
            in[i * 2] = a.steps[i].accel;
            in[i * 2 + 1] = a.steps[i].curvature;
        }
        check(alpa_rollout(ctx_, in.data(), 1, initial_speed, out.data()), ctx_);
        Trajectory t;
        t.poses.resize(static_cast<size_t>(A));
        for (std::int64_t i = 0; i < A; ++i) t.poses[i] = {out[i * 3], out[i * 3 + 1], out[i * 3 + 2]};
        return t;
    }

    // minivla::min_ade / minivla::diversity (eval.cpp:39-59) on the device, bit-exact.
    double min_ade(const std::vector<Trajectory>& samples, const Trajectory& gt) {
        std::vector<float> t = flatten(samples), g = flatten({gt});
        double out = 0.0;
        check(alpa_eval_open_loop(ctx_, t.data(), g.data(), 1, static_cast<std::int64_t>(samples.size()),
                                  static_cast<std::int64_t>(gt.poses.size()), &out, nullptr),
              ctx_);
        return out;
    }
    double diversity(const std::vector<Trajectory>& samples) {
        std::vector<float> t = flatten(samples);
        const std::int64_t steps = samples.empty() ? 0 : static_cast<std::int64_t>(samples[0].poses.size());
        double out = 0.0;
        check(alpa_eval_open_loop(ctx_, t.data(), nullptr, 1, static_cast<std::int64_t>(samples.size()), steps,
                                  nullptr, &out),
              ctx_);
        return out;
    }

    // LatencyReport (profiler.hpp:31-46, profiler.cpp:31-46 key set) of the last
    // run_action_generation: the action-generation component and its counters;
    // the reasoning / preprocessing components belong to stages outside this path.
    // Engine::run_reasoning with the language model on the device (SURVEY
    // §8f-1): vision rows [lanes][P][hidden] (the vision encoder's output, f32)
    // and the prompt ids in; prefill + the decode loop of reasoning_pass
    // (pipeline.cpp:279-390) with the reference's sampler; the sealed KV stays
    // in the library, in place, and the returned ReasoningOutput refers to it.
    ReasoningOutput run_reasoning_device(const std::vector<float>& vision_rows, std::int64_t patches,
                                         const std::vector<std::int64_t>& prompt_ids,
                                         const InferenceRequest& request, std::int64_t max_new_tokens = 256,
                                         std::int64_t termination_token = 0) {
        using clk = std::chrono::steady_clock;
        const std::int64_t lanes = request.topology == Topology::Multi ? request.num_trajectories : 1;
        if (lanes < 1) throw ConfigError("num_trajectories must be >= 1");
        const std::int64_t T = patches + static_cast<std::int64_t>(prompt_ids.size());
        const std::int64_t V = cfg_.vocab_size;
        const auto t0 = clk::now();
        check(alpa_reasoning_begin(ctx_, lanes, T + max_new_tokens), ctx_);
        std::vector<float> logits(static_cast<size_t>(lanes * V));
        check(alpa_reasoning_prefill(ctx_, vision_rows.data(), patches, prompt_ids.data(),
                                     static_cast<std::int64_t>(prompt_ids.size()), logits.data()),
              ctx_);
        const auto t1 = clk::now();
        ReasoningOutput out;
        out.cot_tokens.assign(static_cast<size_t>(lanes), {});
        out.prompt_tokens = T;
        std::vector<std::uint64_t> rng(static_cast<size_t>(lanes));
        for (std::int64_t l = 0; l < lanes; ++l) rng[l] = request.sampler_seed + static_cast<std::uint64_t>(l);
        std::vector<bool> done(static_cast<size_t>(lanes), false);
        const bool forced = request.forced_cot_tokens > 0;
        const std::int64_t max_m = forced ? std::min(request.forced_cot_tokens, max_new_tokens) : max_new_tokens;
        std::vector<std::int64_t> ids(static_cast<size_t>(lanes));
        std::int64_t m = 0;
        while (m < max_m) {
            bool all_done = true;
            for (std::int64_t l = 0; l < lanes; ++l) all_done = all_done && done[l];
            if (all_done && !forced) break;
            for (std::int64_t l = 0; l < lanes; ++l) {
                check(alpa_sample_token(logits.data() + l * V, V, request.sampler_mode == SampleMode::Stochastic,
                                        &rng[l], &ids[l]),
                      nullptr);
                if (!done[l]) {
                    if (!forced && ids[l] == termination_token) done[l] = true;
                    else out.cot_tokens[l].push_back(ids[l]);
                }
            }
            m += 1;
            check(alpa_reasoning_decode(ctx_, ids.data(), logits.data()), ctx_);
        }
        out.token_count = m;
        check(alpa_reasoning_seal(ctx_, &out.reasoning_len), ctx_);
        const auto t2 = clk::now();
        out.n_prefix = lanes;
        out.device_resident = true;
        produced_id_ = out.id;
        reasoning_prefill_ms_ = std::chrono::duration<double, std::milli>(t1 - t0).count();
        reasoning_decode_ms_ = std::chrono::duration<double, std::milli>(t2 - t1).count();
        cot_tokens_ = static_cast<std::int64_t>(out.cot_tokens[0].size());
        return out;
    }

    LatencyReport latency_report() const {
        LatencyReport r;
        r.component_ms[2] = reasoning_prefill_ms_;  // LatencyComponent::ReasoningPrefill
        r.component_ms[3] = reasoning_decode_ms_;   // LatencyComponent::ReasoningDecode
        r.cot_tokens = cot_tokens_;
        r.component_ms[4] = last_stats_.device_ms;  // LatencyComponent::ActionGen
        r.total_ms = last_stats_.device_ms + reasoning_prefill_ms_ + reasoning_decode_ms_;
        r.action_gen_iter_ms.assign(last_stats_.iter_ms, last_stats_.iter_ms + last_stats_.n_iter);
        r.alloc_count = 0;  // every buffer is allocated before the first launch
        r.dispatch_count = static_cast<std::uint64_t>(last_stats_.kernel_launches);
        r.replay_count = static_cast<std::uint64_t>(last_stats_.graph_launches);
        r.bytes_allocated = static_cast<std::uint64_t>(last_stats_.bytes_allocated);
        r.kv_bytes = last_stats_.kv_bytes;
        return r;
    }

private:
    alpa_stats last_stats_{};
    std::uint64_t produced_id_ = 0;
    double reasoning_prefill_ms_ = 0.0, reasoning_decode_ms_ = 0.0;
    std::int64_t cot_tokens_ = 0;
    static std::vector<float> flatten(const std::vector<Trajectory>& ts) {
        std::vector<float> out;
        for (const Trajectory& t : ts) {
            if (!ts.empty() && t.poses.size() != ts[0].poses.size())
                throw InternalError("trajectory length mismatch");  // eval.cpp:15-17
            for (const Pose& p : t.poses) {
                out.push_back(p.x);
                out.push_back(p.y);
                out.push_back(p.yaw);
            }
        }
        return out;
    }
    // Rebind unless the SAME content is bound: keyed on the object's id (fresh
    // per ReasoningOutput, so a new object at a reused address rebinds), its
    // version (touch()), the data pointers and the shape.
    void bind(const ReasoningOutput& r) {
        if (r.device_resident) {
            if (r.id != produced_id_)
                throw InternalError("device reasoning output of another engine or an earlier scene");
            return;  // bound by alpa_reasoning_seal
        }
        const BindKey k{r.id, r.version, r.kv_device, r.kv_host.data(), r.kv_host.size(), r.n_prefix,
                        r.reasoning_len};
        if (bound_valid_ && k == bound_) return;
        if (r.kv_device)
            check(alpa_bind_prefix_device(ctx_, r.kv_device, r.n_prefix, r.reasoning_len), ctx_);
        else
            check(alpa_bind_prefix(ctx_, r.kv_host.data(), r.n_prefix, r.reasoning_len), ctx_);
        bound_ = k;
        bound_valid_ = true;
    }
    struct BindKey {
        std::uint64_t id, version;
        const void* dev;
        const float* host;
        size_t host_n;
        std::int64_t n_prefix, r;
        bool operator==(const BindKey& o) const {
            return id == o.id && version == o.version && dev == o.dev && host == o.host &&
                   host_n == o.host_n && n_prefix == o.n_prefix && r == o.r;
        }
    };
    static alpa_request to_c(const InferenceRequest& q) {
        alpa_request r{};
        r.num_trajectories = q.num_trajectories;
        r.lane0 = 0;
        r.action_init_seed = q.action_init_seed;
        r.action_seed_stride = q.action_seed_stride;
        r.diffusion_iters = 0;
        r.topology = q.topology == Topology::Single ? ALPA_TOPOLOGY_SINGLE : ALPA_TOPOLOGY_MULTI;
        r.kv_strategy = q.kv_strategy == KvStrategy::Static ? ALPA_KV_STATIC : ALPA_KV_DYNAMIC;
        r.executor = q.executor == ExecMode::Graph ? ALPA_EXEC_GRAPH : ALPA_EXEC_EAGER;
        r.v0 = initial_speed_from_history(q.pose_history);
        return r;
    }

    ModelConfig cfg_;
    alpa_ctx* ctx_ = nullptr;
    BindKey bound_{};
    bool bound_valid_ = false;
};

}  // namespace alpa_shim
