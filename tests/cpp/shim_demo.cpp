// Reference-style caller of the C++ shim (include/alpa_minivla_shim.hpp): the
// code a minivla user writes around Engine::run_action_generation, unchanged
// except for the namespace.  Used by tests/test_shim.py.
//
//   shim_demo <prefix.bin> <r> <n> <out_actions.bin> <out_traj.bin>
// exit codes follow the reference CLI (cli.cpp:528-540): 1 io, 2 config, 3 internal.
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "alpa_minivla_shim.hpp"

using namespace alpa_shim;

// shim_demo --reason <vision.bin f32 [P][hidden]> <P> <prompt.bin int64> <n> <out_actions.bin> <out_traj.bin>:
// the reasoning stage's language model on the device (Engine::run_reasoning_device),
// then the action stage on the in-place KV, as Engine::infer sequences them.
static int reason_mode(char** argv) {
    ModelConfig cfg;
    Engine engine(cfg);
    const std::int64_t P = std::atoll(argv[3]);
    std::vector<float> vision(static_cast<size_t>(P * cfg.hidden_dim));
    std::ifstream vin(argv[2], std::ios::binary);
    if (!vin.read(reinterpret_cast<char*>(vision.data()), vision.size() * sizeof(float)))
        throw IoError("cannot read vision rows");
    std::ifstream pin(argv[4], std::ios::binary | std::ios::ate);
    if (!pin) throw IoError("cannot read prompt ids");
    std::vector<std::int64_t> prompt(static_cast<size_t>(pin.tellg()) / sizeof(std::int64_t));
    pin.seekg(0);
    pin.read(reinterpret_cast<char*>(prompt.data()), prompt.size() * sizeof(std::int64_t));
    InferenceRequest req;
    req.num_trajectories = std::atoll(argv[5]);
    req.topology = Topology::Single;
    req.kv_strategy = KvStrategy::Static;
    req.executor = ExecMode::Graph;
    for (int j = 0; j < 16; ++j) req.pose_history.poses[j] = {-(15.0f - j) * 5.0f * 0.1f, 0.f, 0.f};
    ReasoningOutput reasoning = engine.run_reasoning_device(vision, P, prompt, req);
    const auto actions = engine.run_action_generation(reasoning, req);
    const float v0 = initial_speed_from_history(req.pose_history);
    std::ofstream oa(argv[6], std::ios::binary), ot(argv[7], std::ios::binary);
    for (const auto& a : actions) {
        oa.write(reinterpret_cast<const char*>(a.steps.data()), a.steps.size() * sizeof(ActionStep));
        const Trajectory t = engine.actions_to_trajectory(a, v0);
        ot.write(reinterpret_cast<const char*>(t.poses.data()), t.poses.size() * sizeof(Pose));
    }
    std::printf("reasoning r=%lld steps=%lld\n", static_cast<long long>(reasoning.reasoning_len),
                static_cast<long long>(reasoning.token_count));
    std::printf("report %s\n", engine.latency_report().to_json().c_str());
    return 0;
}

int main(int argc, char** argv) {
    if (argc == 8 && std::string(argv[1]) == "--reason") {
        try {
            return reason_mode(argv);
        } catch (const IoError& e) {
            std::fprintf(stderr, "io error: %s\n", e.what());
            return 1;
        } catch (const ConfigError& e) {
            std::fprintf(stderr, "config error: %s\n", e.what());
            return 2;
        } catch (const InternalError& e) {
            std::fprintf(stderr, "internal error: %s\n", e.what());
            return 3;
        }
    }
    if (argc != 6) return 1;
    try {
        ModelConfig cfg;  // fixtures/default_config.json model block
        Engine engine(cfg);
        ReasoningOutput reasoning;
        reasoning.reasoning_len = std::atoll(argv[2]);
        const size_t n_kv = static_cast<size_t>(cfg.decoder_blocks) * 2 * reasoning.reasoning_len * cfg.kv_dim;
        reasoning.kv_host.resize(n_kv);
        std::ifstream in(argv[1], std::ios::binary);
        if (!in.read(reinterpret_cast<char*>(reasoning.kv_host.data()), n_kv * sizeof(float)))
            throw IoError("cannot read prefix");
        InferenceRequest req;
        req.num_trajectories = std::atoll(argv[3]);
        req.topology = Topology::Single;
        req.kv_strategy = KvStrategy::Static;
        req.executor = ExecMode::Graph;
        for (int j = 0; j < 16; ++j) req.pose_history.poses[j] = {-(15.0f - j) * 5.0f * 0.1f, 0.f, 0.f};
        DiffusionResult diff;
        std::int64_t kv_bytes = 0;
        const auto actions = engine.run_action_generation(reasoning, req, &diff, &kv_bytes);
        const float v0 = initial_speed_from_history(req.pose_history);
        std::ofstream oa(argv[4], std::ios::binary), ot(argv[5], std::ios::binary);
        for (const auto& a : actions) {
            oa.write(reinterpret_cast<const char*>(a.steps.data()), a.steps.size() * sizeof(ActionStep));
            const Trajectory t = engine.actions_to_trajectory(a, v0);
            ot.write(reinterpret_cast<const char*>(t.poses.data()), t.poses.size() * sizeof(Pose));
        }
        std::vector<Trajectory> trajs;
        for (const auto& a : actions) trajs.push_back(engine.actions_to_trajectory(a, v0));
        if (trajs.size() >= 2)  // open-loop metrics on the device (eval.cpp:39-59)
            std::printf("metrics min_ade=%.17g diversity=%.17g\n", engine.min_ade(trajs, trajs[0]),
                        engine.diversity(trajs));
        std::printf("report %s\n", engine.latency_report().to_json().c_str());
        std::printf("ok graph_commands=%lld kv_bytes=%lld device_ms=%.3f\n",
                    static_cast<long long>(diff.graph_commands), static_cast<long long>(kv_bytes),
                    diff.device_ms);
        return 0;
    } catch (const IoError& e) {
        std::fprintf(stderr, "io error: %s\n", e.what());
        return 1;
    } catch (const ConfigError& e) {
        std::fprintf(stderr, "config error: %s\n", e.what());
        return 2;
    } catch (const InternalError& e) {
        std::fprintf(stderr, "internal error: %s\n", e.what());
        return 3;
    }
}
