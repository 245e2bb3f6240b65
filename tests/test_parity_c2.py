"""bf16 parity at the BENCHMARKED depth.

Expected values: tests/golden/expected_c2.npz, written by
tests/golden/make_golden_c2.py from the C restatement of the reference path
(pinned bitwise to the reference itself at config-2 width, golden_c2.json
"pin").  Shape: Alpamayo-1-width action expert (ah 2048, kv 1024, 8 heads),
r = 2048 synthetic prefix (make_sealed_cache recipe, seed 4242), weight seed
1234, noise seed 2 stride 1, v0 = 5.0.

Bar (BASELINE.json north_star): rel-L2 <= 2e-2 for bf16 tensor-core
trajectories against the CPU oracle; the measured error is printed (and
collected into profiles/ by tools/gpu_round.sh).
"""
import json
import os

import numpy as np
import pytest

import paper_2605_08975_b200 as alpa

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2
HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "expected_c2.npz")
META = os.path.join(HERE, "golden", "golden_c2.json")


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def c2gold():
    g = np.load(GOLD)
    with open(META) as f:
        meta = json.load(f)
    return g, meta


def c2(B, K):
    return alpa.ModelConfig(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=B,
                            action_hidden_dim=2048, kv_dim=1024, heads=8, diffusion_iters=K,
                            dtype="bf16")


def _record(name, err_a, err_t):
    line = json.dumps({"case": name, "rel_l2_actions": err_a, "rel_l2_traj": err_t})
    print(line)
    out = os.environ.get("ALPA_PARITY_LOG")
    if out:
        with open(out, "a") as f:
            f.write(line + "\n")


@pytest.mark.parametrize("name", ["c2_n6_k10", "c2_n1_k10", "b2_n64_k2", "b1_n6_k5", "b1_n6_k20"])
def test_bf16_parity_benchmarked_depth(c2gold, name):
    g, meta = c2gold
    case = meta["cases"][name]
    m = c2(case["B"], case["K"])
    with alpa.ActionGenerator(m) as gen:
        gen.bind_prefix_synthetic(meta["prefix_seed"], meta["r"])
        res = gen.run_action_generation(alpa.InferenceRequest(num_trajectories=case["n"],
                                                              v0=meta["v0"]))
    ea, et = rel_l2(res.actions, g[f"{name}_actions"]), rel_l2(res.trajectories, g[f"{name}_traj"])
    _record(name, ea, et)
    assert ea <= BF16_TOL
    assert et <= BF16_TOL


def test_bf16_parity_multi_topology(c2gold):
    """Multi topology (lane l attends prefix l, pipeline.cpp:405-413) at
    config-2 width: three distinct synthesized prefixes bound on the device."""
    torch = pytest.importorskip("torch")
    g, meta = c2gold
    name = "multi_n3_b2_k2"
    case = meta["cases"][name]
    m = c2(case["B"], case["K"])
    n = case["n"]
    with alpa.ActionGenerator(m) as gen:
        per = gen.prefix_bytes(meta["r"])
        buf = torch.empty(n * per, dtype=torch.uint8, device="cuda")
        for l in range(n):
            gen.synthesize_prefix(buf.data_ptr() + l * per, meta["prefix_seed"] + 1000 * l, meta["r"])
        torch.cuda.synchronize()
        gen.bind_prefix_device(buf.data_ptr(), n, meta["r"])
        res = gen.run_action_generation(alpa.InferenceRequest(num_trajectories=n, topology="multi",
                                                              v0=meta["v0"]))
        del buf
    ea, et = rel_l2(res.actions, g[f"{name}_actions"]), rel_l2(res.trajectories, g[f"{name}_traj"])
    _record(name, ea, et)
    assert ea <= BF16_TOL
    assert et <= BF16_TOL
