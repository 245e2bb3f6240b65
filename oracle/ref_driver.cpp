// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Thin extern "C" driver around the UNMODIFIED reference sources
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libminivla_ref.so).  It exposes exactly the reference calls the
// hot path needs so Python tests / bench can drive the real reference:
//   * ref_scenario_prefix   — Engine::run_reasoning on a scenario
//                             (pipeline.cpp:393-397), returning the sealed
//                             prefix KV of lane 0 as [B][2][r][kv] f32 and
//                             KvCache::reasoning_fingerprint (kv_cache.cpp:346)
//   * ref_action_generation — Engine::run_action_generation
//                             (pipeline.cpp:399-436) on a caller-supplied
//                             prefix, timed exactly like cli.cpp:273-278
//   * ref_rollout           — actions_to_trajectory (pipeline.cpp:124-148)
//   * ref_action_weights    — ModelWeights::build (model.cpp:120-151) action
//                             tensors, to pin the weight-stream restatement
// No reference source is copied here; everything is a call into it.

#include "minivla/common.hpp"
#include "minivla/eval.hpp"
#include "minivla/profiler.hpp"
#include "minivla/kv_cache.hpp"
#include "minivla/model.hpp"
#include "minivla/pipeline.hpp"
#include "minivla/scenario.hpp"

#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <span>
#include <vector>

using namespace minivla;

namespace {
thread_local std::string g_err;

int fail(const Error& e, int code) {
    g_err = e.what();
    return code;
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const IoError& e) {
        return fail(e, 1);
    } catch (const ConfigError& e) {
        return fail(e, 2);
    } catch (const InternalError& e) {
        return fail(e, 3);
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}
} // namespace

extern "C" {

// Field order is mirrored by oracle/_refdrv.py (ctypes).
struct RefCfg {
    std::int64_t vision_blocks;
    std::int64_t decoder_blocks;
    std::int64_t hidden_dim;
    std::int64_t action_hidden_dim;
    std::int64_t kv_dim;
    std::int64_t heads;
    std::int64_t vocab_size;
    std::int64_t patch_size;
    std::int64_t action_steps;
    std::int64_t diffusion_iters;
    std::int64_t max_new_tokens;
    float update_scale;
    std::uint64_t weight_seed;
};

static ModelConfig to_cfg(const RefCfg* c) {
    ModelConfig m;
    m.vision_blocks = c->vision_blocks;
    m.decoder_blocks = c->decoder_blocks;
    m.hidden_dim = c->hidden_dim;
    m.action_hidden_dim = c->action_hidden_dim;
    m.kv_dim = c->kv_dim;
    m.heads = c->heads;
    m.vocab_size = c->vocab_size;
    m.patch_size = c->patch_size;
    m.action_steps = c->action_steps;
    m.diffusion_iters = c->diffusion_iters;
    m.max_new_tokens = c->max_new_tokens;
    m.update_scale = c->update_scale;
    m.weight_seed = c->weight_seed;
    return m;
}

const char* ref_last_error() { return g_err.c_str(); }

// Reasoning stage on a scenario file (single topology, batch-1 prefix).
// out may be null (size query): r_out receives the prefix length.
int ref_scenario_prefix(const RefCfg* c, const char* scenario_path,
                        std::uint64_t sampler_seed, int stochastic,
                        std::int64_t forced_cot, int static_kv, float* out,
                        std::int64_t out_capacity, std::int64_t* r_out,
                        std::uint64_t* fingerprint_out, float* v0_out) {
    return guarded([&] {
        const ModelConfig cfg = to_cfg(c);
        Engine engine(cfg);
        RunConfig rc;
        rc.model = cfg;
        const Scenario sc = load_scenario(scenario_path);
        InferenceRequest req = request_from_scenario(sc, rc);
        req.topology = Topology::Single;
        req.num_trajectories = 1;
        req.kv_strategy = static_kv ? KvStrategy::Static : KvStrategy::Dynamic;
        req.executor = ExecMode::Eager;
        req.sampler_seed = sampler_seed;
        req.sampler_mode = stochastic ? SampleMode::Stochastic : SampleMode::Greedy;
        req.forced_cot_tokens = forced_cot;
        ReasoningOutput ro = engine.run_reasoning(req);
        const std::int64_t r = ro.kv.reasoning_len();
        const std::int64_t kd = cfg.kv_dim;
        const std::int64_t B = cfg.decoder_blocks;
        if (r_out) *r_out = r;
        if (fingerprint_out) *fingerprint_out = ro.kv.reasoning_fingerprint();
        if (v0_out) *v0_out = initial_speed_from_history(req.pose_history);
        if (!out) return;
        if (out_capacity < B * 2 * r * kd) throw InternalError("prefix buffer too small");
        for (std::int64_t b = 0; b < B; ++b) {
            const auto data = engine.substrate().read(ro.kv.block_buffer(b));
            const std::int64_t cap = engine.substrate().shape(ro.kv.block_buffer(b))[2];
            for (int s = 0; s < 2; ++s) {
                // [2][batch=1][cap][kv] -> [B][2][r][kv]
                std::memcpy(out + ((b * 2 + s) * r) * kd, data.data() + (s * cap) * kd,
                            static_cast<std::size_t>(r * kd) * sizeof(float));
            }
        }
    });
}

// Inputs and outputs of the reasoning stage on a scenario (single topology),
// for the device KV producer's parity test: the vision encoder's rows
// (Model::vision_encode, model.cpp:326-392, on the request's patch rows as in
// pipeline.cpp:265-277) [P][hidden], the prompt token ids
// (Engine::preprocess), and the ids the decode loop fed back
// (Engine::run_reasoning: cot tokens, plus the terminator when the loop
// stopped on it, pipeline.cpp:345-386); T = P + prompt, m = decode steps.
// Null outputs: size query.
int ref_reasoning_io(const RefCfg* c, const char* scenario_path, std::uint64_t sampler_seed,
                     int stochastic, float* vision_out, std::int64_t vision_cap,
                     std::int64_t* P_out, std::int64_t* prompt_out, std::int64_t prompt_cap,
                     std::int64_t* n_prompt_out, std::int64_t* ids_out, std::int64_t ids_cap,
                     std::int64_t* m_out, std::int64_t* T_out) {
    return guarded([&] {
        const ModelConfig cfg = to_cfg(c);
        Engine engine(cfg);
        RunConfig rc;
        rc.model = cfg;
        const Scenario sc = load_scenario(scenario_path);
        InferenceRequest req = request_from_scenario(sc, rc);
        req.topology = Topology::Single;
        req.num_trajectories = 1;
        req.kv_strategy = KvStrategy::Static;
        req.executor = ExecMode::Eager;
        req.sampler_seed = sampler_seed;
        req.sampler_mode = stochastic ? SampleMode::Stochastic : SampleMode::Greedy;
        const Engine::Preprocessed pre = engine.preprocess(req);
        Substrate& sub = engine.substrate();
        const BufferId patch = sub.alloc({pre.patches, pre.patch_dim});
        sub.write(patch, pre.patch_rows);
        const BufferId vis = engine.model().vision_encode(patch, 1, pre.patches);
        const auto v = sub.read(vis);
        const std::int64_t np = static_cast<std::int64_t>(pre.prompt.ids.size());
        ReasoningOutput ro = engine.run_reasoning(req);
        std::vector<std::int64_t> ids = ro.cot_tokens[0];
        if (static_cast<std::int64_t>(ids.size()) < ro.token_count)
            ids.push_back(engine.tokenizer().termination_token());
        if (P_out) *P_out = pre.patches;
        if (n_prompt_out) *n_prompt_out = np;
        if (m_out) *m_out = ro.token_count;
        if (T_out) *T_out = pre.patches + np;
        if (vision_out) {
            if (vision_cap < static_cast<std::int64_t>(v.size())) throw InternalError("vision buffer too small");
            std::memcpy(vision_out, v.data(), v.size() * sizeof(float));
        }
        if (prompt_out) {
            if (prompt_cap < np) throw InternalError("prompt buffer too small");
            for (std::int64_t i = 0; i < np; ++i) prompt_out[i] = pre.prompt.ids[i];
        }
        if (ids_out) {
            if (ids_cap < static_cast<std::int64_t>(ids.size())) throw InternalError("ids buffer too small");
            for (std::size_t i = 0; i < ids.size(); ++i) ids_out[i] = ids[i];
        }
    });
}

// Engine::run_action_generation on a batch-1 prefix [B][2][r][kv] f32.
// topology_single: 1 = Single (replicate_for_batch when n>1); 0 = Multi
// (prefix replicated by the caller into batch n: prefix is [B][2][n][r][kv]).
// ms_out: wall time of run_action_generation (cli.cpp:273-278 region).
int ref_action_generation(const RefCfg* c, const float* prefix, std::int64_t r,
                          std::int64_t n, std::uint64_t seed, std::uint64_t stride,
                          int static_kv, int graph_exec, int topology_single,
                          int parallel_kernels, float* actions_out, double* ms_out,
                          std::int64_t* kv_bytes_out, double* iter_ms_sum_out) {
    return guarded([&] {
        const ModelConfig cfg = to_cfg(c);
        SubstrateOptions so;
        so.parallel_kernels = parallel_kernels != 0;
        Engine engine(cfg, so);
        Substrate& sub = engine.substrate();
        const std::int64_t kd = cfg.kv_dim;
        const std::int64_t B = cfg.decoder_blocks;
        const std::int64_t batch = topology_single ? 1 : n;
        KvLayout lay;
        lay.num_blocks = B;
        lay.batch = batch;
        lay.kv_dim = kd;
        lay.action_len = cfg.action_steps;
        lay.reasoning_capacity = r;
        KvCache kv(sub, static_kv ? KvStrategy::Static : KvStrategy::Dynamic, lay);
        for (std::int64_t b = 0; b < B; ++b) {
            std::vector<float> kbuf(batch * r * kd), vbuf(batch * r * kd);
            for (std::int64_t l = 0; l < batch; ++l) {
                const float* src = prefix + ((b * 2) * batch + l) * r * kd;
                const float* srcv = prefix + ((b * 2 + 1) * batch + l) * r * kd;
                std::memcpy(kbuf.data() + l * r * kd, src, r * kd * sizeof(float));
                std::memcpy(vbuf.data() + l * r * kd, srcv, r * kd * sizeof(float));
            }
            const BufferId kb = sub.alloc({batch * r, kd});
            const BufferId vb = sub.alloc({batch * r, kd});
            sub.write(kb, kbuf);
            sub.write(vb, vbuf);
            kv.append_reasoning(b, kb, vb, r);
        }
        kv.seal_reasoning();
        ReasoningOutput ro{{}, 0, r, std::move(kv), kInvalidBuffer};
        InferenceRequest req;
        req.num_trajectories = n;
        req.topology = topology_single ? Topology::Single : Topology::Multi;
        req.kv_strategy = static_kv ? KvStrategy::Static : KvStrategy::Dynamic;
        req.executor = graph_exec ? ExecMode::Graph : ExecMode::Eager;
        req.action_init_seed = seed;
        req.action_seed_stride = stride;
        Model::DiffusionResult diff;
        std::int64_t kv_bytes = 0;
        const auto t0 = std::chrono::steady_clock::now();
        const auto actions = engine.run_action_generation(ro, req, &diff, &kv_bytes);
        const double ms = std::chrono::duration<double, std::milli>(
                              std::chrono::steady_clock::now() - t0)
                              .count();
        if (ms_out) *ms_out = ms;
        // DiffusionResult::iter_ms (model.hpp:155-160): the K refinement
        // iterations alone; the rest of the region is noise + replicate_for_batch
        if (iter_ms_sum_out) {
            double s = 0.0;
            for (double v : diff.iter_ms) s += v;
            *iter_ms_sum_out = s;
        }
        if (kv_bytes_out) *kv_bytes_out = kv_bytes;
        for (std::int64_t l = 0; l < n; ++l) {
            for (std::int64_t i = 0; i < cfg.action_steps; ++i) {
                actions_out[(l * cfg.action_steps + i) * 2] = actions[l].steps[i].accel;
                actions_out[(l * cfg.action_steps + i) * 2 + 1] =
                    actions[l].steps[i].curvature;
            }
        }
    });
}

// actions [n][64][2] -> traj [n][64][3] via the reference rollout.
int ref_rollout(const float* actions, std::int64_t n, float v0, float* traj_out) {
    return guarded([&] {
        for (std::int64_t l = 0; l < n; ++l) {
            ActionSequence a;
            a.steps.resize(64);
            for (int i = 0; i < 64; ++i) {
                a.steps[i] = {actions[(l * 64 + i) * 2], actions[(l * 64 + i) * 2 + 1]};
            }
            const Trajectory t = actions_to_trajectory(a, v0);
            for (int i = 0; i < 64; ++i) {
                traj_out[(l * 64 + i) * 3] = t.poses[i].x;
                traj_out[(l * 64 + i) * 3 + 1] = t.poses[i].y;
                traj_out[(l * 64 + i) * 3 + 2] = t.poses[i].yaw;
            }
        }
    });
}

// Copies one action-expert tensor drawn by ModelWeights::build.
// which: 0 action_in.w, 1 action_in.b, 2 mlp1.w, 3 mlp1.b, 4 mlp2.w, 5 mlp2.b,
// 6 head.w, 7 head.b, 10+6*blk+{0..5}*? -> per block: (q,k,v,o,mlp1,mlp2)
// encoded as 100 + blk*20 + lin*2 + (0 w | 1 b).
int ref_action_weights(const RefCfg* c, int which, float* out, std::int64_t cap,
                       std::int64_t* count_out) {
    return guarded([&] {
        const ModelWeights w = ModelWeights::build(to_cfg(c));
        const std::vector<float>* src = nullptr;
        auto pick = [&](const LinearWeights& l, int wb) { src = wb ? &l.b : &l.w; };
        if (which < 100) {
            switch (which) {
            case 0: src = &w.action_in.w; break;
            case 1: src = &w.action_in.b; break;
            case 2: src = &w.action_mlp1.w; break;
            case 3: src = &w.action_mlp1.b; break;
            case 4: src = &w.action_mlp2.w; break;
            case 5: src = &w.action_mlp2.b; break;
            case 6: src = &w.action_head.w; break;
            case 7: src = &w.action_head.b; break;
            default: throw ConfigError("bad tensor id");
            }
        } else {
            const int blk = (which - 100) / 20;
            const int lin = ((which - 100) % 20) / 2;
            const int wb = (which - 100) % 2;
            const BlockWeights& bw = w.action.at(blk);
            const LinearWeights* ls[6] = {&bw.q, &bw.k, &bw.v, &bw.o, &bw.mlp1, &bw.mlp2};
            if (lin > 5) throw ConfigError("bad tensor id");
            pick(*ls[lin], wb);
        }
        *count_out = static_cast<std::int64_t>(src->size());
        if (out) {
            if (cap < *count_out) throw InternalError("buffer too small");
            std::memcpy(out, src->data(), src->size() * sizeof(float));
        }
    });
}

// LatencyReport::from_json of the reference on a JSON document (wire-format
// check of the shim's report); writes back the number of iteration entries.
int ref_parse_latency_report(const char* json, std::int64_t* n_iter, double* action_gen_ms) {
    return guarded([&] {
        const LatencyReport r = LatencyReport::from_json(nlohmann::json::parse(json));
        *n_iter = static_cast<std::int64_t>(r.action_gen_iter_ms.size());
        *action_gen_ms = r.component_ms[static_cast<int>(LatencyComponent::ActionGen)];
    });
}

// minivla::min_ade / minivla::diversity (eval.cpp:39-59) on [n][64][3] poses.
static std::vector<Trajectory> to_trajs(const float* traj, std::int64_t n, std::int64_t steps) {
    std::vector<Trajectory> out(static_cast<std::size_t>(n));
    for (std::int64_t l = 0; l < n; ++l) {
        out[l].poses.resize(steps);
        for (std::int64_t i = 0; i < steps; ++i)
            out[l].poses[i] = {traj[(l * steps + i) * 3], traj[(l * steps + i) * 3 + 1],
                               traj[(l * steps + i) * 3 + 2]};
    }
    return out;
}
int ref_min_ade(const float* traj, std::int64_t n, std::int64_t steps, const float* gt, double* out) {
    return guarded([&] {
        const std::vector<Trajectory> s = to_trajs(traj, n, steps);
        const std::vector<Trajectory> g = to_trajs(gt, 1, steps);
        *out = min_ade(std::span<const Trajectory>(s), g[0]);
    });
}
int ref_diversity(const float* traj, std::int64_t n, std::int64_t steps, double* out) {
    return guarded([&] {
        const std::vector<Trajectory> s = to_trajs(traj, n, steps);
        *out = diversity(std::span<const Trajectory>(s));
    });
}

} // extern "C"
