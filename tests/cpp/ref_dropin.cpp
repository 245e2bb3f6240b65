// Drop-in test: the REFERENCE engine (minivla, compiled from /root/reference
// sources by oracle/Makefile) with its action stage routed to the B200 library
// through include/alpa_minivla_adapter.hpp -- the reference's own types end to
// end (ReasoningOutput, InferenceRequest, ActionSequence, Trajectory).
//
// For each topology x N x variant of cmd_compare_actiongen (cli.cpp:236-313:
// dynamic/eager, static/eager, static/graph):
//   reference : Engine::infer(req)                        (pipeline.cpp:438-500)
//   drop-in   : Engine::run_reasoning(req) -> ActionStage::run_action_generation
//               -> minivla::actions_to_trajectory (host, reference code)
// and checks actions / trajectories rel-L2 <= 1e-4 (fp32 path), the device
// rollout == the reference's host rollout bitwise, every variant bitwise equal
// to the first (cli.cpp:292-300), kv_bytes == LatencyReport::kv_bytes, and the
// reference's error types for N = 0 and graph + dynamic.
//
// Plus the reasoning stage on the device (ActionStage::run_reasoning, SURVEY
// §8f-1): chain-of-thought tokens equal to Engine::run_reasoning's, and
// actions / trajectories off the in-place device KV vs Engine::infer.
//
// Prints one JSON line per case; exit 0 all pass, 3 a failure (cli.cpp:528-540).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <minivla/pipeline.hpp>
#include <minivla/scenario.hpp>

#include "alpa_minivla_adapter.hpp"

using namespace minivla;

namespace {

double rel_l2(const std::vector<float>& a, const std::vector<float>& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        const double d = (double)a[i] - (double)b[i];
        num += d * d;
        den += (double)b[i] * b[i];
    }
    return std::sqrt(num) / std::max(std::sqrt(den), 1e-30);
}
std::vector<float> flat(const std::vector<ActionSequence>& v) {
    std::vector<float> o;
    for (const auto& s : v)
        for (const auto& st : s.steps) {
            o.push_back(st.accel);
            o.push_back(st.curvature);
        }
    return o;
}
std::vector<float> flat(const std::vector<Trajectory>& v) {
    std::vector<float> o;
    for (const auto& t : v)
        for (const auto& p : t.poses) {
            o.push_back(p.x);
            o.push_back(p.y);
            o.push_back(p.yaw);
        }
    return o;
}

// A demo-like scenario built in code (the reference's own procedural frames,
// a straight 5 m/s history, the RunConfig default prompts).
Scenario make_scenario() {
    Scenario s;
    s.frames = synthetic_frames(56, 56, "gradient");
    for (int i = 0; i < 16; ++i) s.past_poses.poses[i] = Pose{-7.5f + 0.5f * (float)i, 0.0f, 0.0f};
    RunConfig rc;
    s.system_prompt = rc.default_system_prompt;
    s.user_prompt = rc.default_user_prompt;
    return s;
}

}  // namespace

int main(int argc, char** argv) {
    const int device = argc > 1 ? std::atoi(argv[1]) : 0;
    bool ok = true;
    try {
        RunConfig rc;  // model = ModelConfig defaults (model.hpp:12-29)
        const Scenario sc = make_scenario();
        Engine engine(rc.model, rc.substrate_options());
        alpa_minivla::ActionStage gpu(rc.model, device);
        struct Variant {
            const char* name;
            KvStrategy kv;
            ExecMode mode;
        };
        const Variant variants[] = {{"baseline", KvStrategy::Dynamic, ExecMode::Eager},
                                    {"+static_kv", KvStrategy::Static, ExecMode::Eager},
                                    {"+graph", KvStrategy::Static, ExecMode::Graph}};
        for (Topology topo : {Topology::Single, Topology::Multi}) {
            for (std::int64_t n : {1, 6}) {
                std::vector<float> first_traj;
                for (const Variant& v : variants) {
                    RunConfig c = rc;
                    c.topology = topo;
                    c.num_trajectories = n;
                    c.kv_strategy = v.kv;
                    c.executor = v.mode;
                    InferenceRequest req = request_from_scenario(sc, c);
                    const InferenceResult ref = engine.infer(req);
                    ReasoningOutput reasoning = engine.run_reasoning(req);
                    Model::DiffusionResult diff;
                    std::int64_t kvb = 0;
                    const auto acts = gpu.run_action_generation(engine.substrate(), reasoning, req, &diff, &kvb);
                    const float v0 = initial_speed_from_history(req.pose_history);
                    std::vector<Trajectory> traj;
                    bool rollout_bitexact = true;
                    for (const auto& a : acts) {
                        traj.push_back(actions_to_trajectory(a, v0));  // the reference's host rollout
                        const Trajectory dt = gpu.actions_to_trajectory(a, v0);
                        rollout_bitexact = rollout_bitexact &&
                                           std::memcmp(dt.poses.data(), traj.back().poses.data(),
                                                       dt.poses.size() * sizeof(Pose)) == 0;
                    }
                    const double ea = rel_l2(flat(acts), flat(ref.actions));
                    const double et = rel_l2(flat(traj), flat(ref.trajectories));
                    const auto ft = flat(traj);
                    const bool same = first_traj.empty() || first_traj == ft;
                    if (first_traj.empty()) first_traj = ft;
                    const bool pass = ea <= 1e-4 && et <= 1e-4 && rollout_bitexact && same &&
                                      kvb == ref.latency.kv_bytes && (int64_t)acts.size() == n &&
                                      (int64_t)diff.iter_ms.size() == rc.model.diffusion_iters;
                    ok = ok && pass;
                    std::printf(
                        "{\"topology\": \"%s\", \"n\": %lld, \"variant\": \"%s\", \"rel_l2_actions\": %.3e, "
                        "\"rel_l2_traj\": %.3e, \"device_rollout_bitexact\": %s, \"variants_equal\": %s, "
                        "\"kv_bytes\": %lld, \"ref_kv_bytes\": %lld, \"pass\": %s}\n",
                        topo == Topology::Single ? "single" : "multi", (long long)n, v.name, ea, et,
                        rollout_bitexact ? "true" : "false", same ? "true" : "false", (long long)kvb,
                        (long long)ref.latency.kv_bytes, pass ? "true" : "false");
                }
            }
        }
        // the reasoning stage on the device: the reference engine keeps
        // vision + tokenizer; the LM's prefill/decode and the KV run in the library and
        // the action stage attends the KV in place -- vs Engine::infer end to end
        for (Topology topo : {Topology::Single, Topology::Multi}) {
            for (std::int64_t n : {1, 6}) {
                RunConfig c = rc;
                c.topology = topo;
                c.num_trajectories = n;
                c.kv_strategy = KvStrategy::Static;
                c.executor = ExecMode::Graph;
                InferenceRequest req = request_from_scenario(sc, c);
                const InferenceResult ref = engine.infer(req);
                ReasoningOutput refr = engine.run_reasoning(req);
                const auto dr = gpu.run_reasoning(engine, req);
                const auto acts = gpu.run_action_generation_device(req);
                const float v0 = initial_speed_from_history(req.pose_history);
                std::vector<Trajectory> traj;
                for (const auto& a : acts) traj.push_back(actions_to_trajectory(a, v0));
                const double ea = rel_l2(flat(acts), flat(ref.actions));
                const double et = rel_l2(flat(traj), flat(ref.trajectories));
                const bool tokens_equal = dr.cot_tokens == refr.cot_tokens && dr.token_count == refr.token_count;
                const bool len_equal = dr.reasoning_len == refr.kv.reasoning_len();
                const bool pass = ea <= 1e-4 && et <= 1e-4 && tokens_equal && len_equal;
                ok = ok && pass;
                std::printf(
                    "{\"device_reasoning\": true, \"topology\": \"%s\", \"n\": %lld, \"r\": %lld, "
                    "\"tokens_equal\": %s, \"rel_l2_actions\": %.3e, \"rel_l2_traj\": %.3e, \"pass\": %s}\n",
                    topo == Topology::Single ? "single" : "multi", (long long)n, (long long)dr.reasoning_len,
                    tokens_equal ? "true" : "false", ea, et, pass ? "true" : "false");
            }
        }
        // the reference's error types through the adapter
        InferenceRequest req = request_from_scenario(sc, rc);
        ReasoningOutput reasoning = engine.run_reasoning(req);
        auto expect = [&](const char* what, auto fn, bool want_config) {
            bool got = false;
            try {
                fn();
            } catch (const ConfigError&) {
                got = want_config;
            } catch (const InternalError&) {
                got = !want_config;
            }
            ok = ok && got;
            std::printf("{\"error_case\": \"%s\", \"pass\": %s}\n", what, got ? "true" : "false");
        };
        expect("n=0 -> InternalError (pipeline.cpp:411-413)", [&] {
            InferenceRequest r = req;
            r.num_trajectories = 0;
            gpu.run_action_generation(engine.substrate(), reasoning, r);
        }, false);
        expect("multi, batch-1 cache, n=3 -> InternalError (pipeline.cpp:411-413)", [&] {
            InferenceRequest r = req;
            r.topology = Topology::Multi;
            r.num_trajectories = 3;
            gpu.run_action_generation(engine.substrate(), reasoning, r);
        }, false);
        expect("graph + dynamic -> ConfigError (model.cpp:609-611)", [&] {
            InferenceRequest r = req;
            r.executor = ExecMode::Graph;
            r.kv_strategy = KvStrategy::Dynamic;
            gpu.run_action_generation(engine.substrate(), reasoning, r);
        }, true);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ref_dropin: %s\n", e.what());
        return 3;
    }
    return ok ? 0 : 3;
}
