"""Regenerate tests/golden/ from the reference itself.

Runs ONLY in the dev container (needs /root/reference, built into
oracle/_ref/libminivla_ref.so by `make -C oracle`).  The outputs are small
committed fixtures so the GPU box (no /root/reference) can check parity:

* prefix_demo.npy      config-1 prefix KV [6][2][427][32] f32: the reference's
                       reasoning stage (Engine::run_reasoning, pipeline.cpp:393)
                       on fixtures/demo_scenario.json, single topology,
                       stochastic sampler seed 1.
* expected_c1.npz      reference actions / trajectories for N in {1,6,16} at
                       K=10, seed 2 stride 1 (Engine::run_action_generation,
                       pipeline.cpp:399-436; actions_to_trajectory,
                       pipeline.cpp:124-148), plus N=6 at K=1 and K=5.
* golden.json          digests (FNV-1a, common.hpp:63-76) and scalars.

Usage:  python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Cfg, Port, Ref  # noqa: E402

SCENARIO = "/root/reference/proj/fixtures/demo_scenario.json"


def main():
    ref, port = Ref(), Port()
    cfg = Cfg.make()  # fixtures/default_config.json model block
    prefix, fingerprint, v0 = ref.scenario_prefix(cfg, SCENARIO)
    np.save(os.path.join(HERE, "prefix_demo.npy"), prefix)
    out = {}
    golden = {"config": cfg.as_dict(), "r": int(prefix.shape[2]),
              "reasoning_fingerprint": f"{fingerprint:016x}", "v0": v0,
              "stream_offset": port.stream_offset(cfg), "runs": {}}
    for n, k in ((1, 10), (6, 10), (16, 10), (6, 1), (6, 5)):
        c = Cfg.make(diffusion_iters=k)
        acts, ms, kvb = ref.action_generation(c, prefix, n)
        traj = ref.rollout(acts, v0)
        key = f"n{n}_k{k}"
        out[f"{key}_actions"] = acts
        out[f"{key}_traj"] = traj
        golden["runs"][key] = {"actions_fnv": f"{port.fnv1a(acts):016x}",
                               "traj_fnv": f"{port.fnv1a(traj):016x}", "kv_bytes": kvb}
    out["noise_n16"] = port.noise(2, 1, 16)
    np.savez_compressed(os.path.join(HERE, "expected_c1.npz"), **out)
    # pins of the weight stream against ModelWeights::build itself
    pins = {}
    for name, which in (("action_in_w", 0), ("head_b", 7), ("blk5_mlp2_b", 100 + 5 * 20 + 5 * 2 + 1),
                        ("blk0_q_w", 100)):
        v = ref.action_weight(cfg, which)
        pins[name] = {"n": int(v.size), "fnv": f"{port.fnv1a(v):016x}",
                      "first": [float(x) for x in v[:4]]}
    golden["weight_pins"] = pins
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(golden, f, indent=1, sort_keys=True)
    print(json.dumps(golden["runs"], indent=1))


if __name__ == "__main__":
    main()
