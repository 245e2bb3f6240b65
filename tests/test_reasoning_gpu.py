"""The on-device reasoning-stage KV producer against the
reference's own reasoning stage on the demo scenario (config 1, fixture
tests/golden/reasoning_c1.npz from tests/golden/make_golden_reasoning.py):

* prefill + teacher-forced decode write the reference's sealed prefix KV, in
  place, in the action stage's layout (rel-L2 <= 1e-4, f32 path);
* the free-running decode loop with the reference's host sampler reproduces the
  reference's chain-of-thought ids exactly (r = 427 = 328 + 99);
* action generation straight off the in-place prefix (capacity stride != r)
  reproduces the reference's Engine actions / trajectories (golden config 1);
* bf16 context: the action-stage copy is the bf16 rounding of the f32 cache,
  and action generation on the in-place prefix equals generation on a compact
  copy of it bitwise (persistent tensor-core kernel); multi topology lanes.
"""
import os

import numpy as np
import pytest

import paper_2605_08975_b200 as alpa

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
F32_TOL = 1e-4


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "reasoning_c1.npz"))


def device_prefix(g, lanes, B, cap, kv, r, dtype="f32"):
    """The bound (in-place) prefix, device -> host: [lanes][B][2][cap][kv],
    live tokens [:r] (f32 values; bf16 contexts widened exactly)."""
    import torch
    from cuda.bindings import runtime as rt

    ptr, nbytes = g.prefix_device()
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    raw = torch.empty(nbytes // (4 if dtype == "f32" else 2), dtype=tdt, device="cuda")
    torch.cuda.synchronize()
    (err,) = rt.cudaMemcpy(raw.data_ptr(), ptr, nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
    assert int(err) == 0, err
    out = raw.float().cpu().numpy().reshape(lanes, B, 2, cap, kv)
    return out[:, :, :, :r, :]


def test_prefill_and_forced_decode_write_the_reference_prefix(gold):
    m = alpa.ModelConfig()  # fixtures/default_config.json model (config 1, f32)
    T, steps = int(gold["T"]), int(gold["m"])
    with alpa.ActionGenerator(m) as g:
        out = g.run_reasoning(gold["vision"], gold["prompt"], forced_ids=gold["decode_ids"])
        assert out["r"] == int(gold["r"]) == T + steps
        cap = T + 256
        got = device_prefix(g, 1, m.decoder_blocks, cap, m.kv_dim, out["r"])[0]
    err = rel_l2(got, gold["prefix"])
    print(f"device prefill+decode KV vs reference: rel-L2 {err:.3e}")
    assert err <= F32_TOL


def test_free_running_decode_reproduces_reference_tokens_and_actions(gold):
    m = alpa.ModelConfig()
    exp = dict(np.load(os.path.join(GOLD, "expected_c1.npz")))
    with alpa.ActionGenerator(m) as g:
        out = g.run_reasoning(gold["vision"], gold["prompt"], sampler_seed=1, stochastic=True)
        ids = list(out["cot_tokens"][0])
        if len(ids) < out["token_count"]:
            ids.append(0)
        assert ids == [int(x) for x in gold["decode_ids"]]
        assert out["r"] == int(gold["r"])
        # the action stage attends the in-place prefix (stride = capacity, r live tokens)
        res = g.run_action_generation(alpa.InferenceRequest(num_trajectories=6, v0=float(gold["v0"])))
    ea = rel_l2(res.actions, exp["n6_k10_actions"])
    et = rel_l2(res.trajectories, exp["n6_k10_traj"])
    print(f"actions off the device-produced prefix vs reference Engine: {ea:.3e} / traj {et:.3e}")
    assert ea <= F32_TOL and et <= F32_TOL


def _bf16_cfg(dtype):
    return alpa.ModelConfig(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=2,
                            action_hidden_dim=256, kv_dim=128, heads=2, diffusion_iters=2, dtype=dtype)


def test_bf16_in_place_prefix_equals_compact_copy():
    """bf16 context: the LM runs in f32 (its own f32 cache); the action-stage
    copy is its bf16 rounding.  Generation on the in-place prefix (capacity
    stride, persistent tensor-core kernel) equals generation on a compact copy
    bitwise, for single and multi topology."""
    import torch
    rng = np.random.default_rng(3)
    vis = (rng.standard_normal((40, 64)) * 0.5).astype(np.float32)
    prompt = rng.integers(1, 128, 25)
    lanes = 3
    with alpa.ActionGenerator(_bf16_cfg("f32")) as g32:
        o32 = g32.run_reasoning(vis, prompt, lanes=lanes, max_new_tokens=40, sampler_seed=11)
        T = 65
        cap = T + 40
        k32 = device_prefix(g32, lanes, 2, cap, 128, o32["r"])
    with alpa.ActionGenerator(_bf16_cfg("bf16")) as g:
        ob = g.run_reasoning(vis, prompt, lanes=lanes, max_new_tokens=40, sampler_seed=11)
        assert ob["cot_tokens"] == o32["cot_tokens"] and ob["r"] == o32["r"]
        kb = device_prefix(g, lanes, 2, cap, 128, ob["r"], dtype="bf16")
        want = torch.from_numpy(k32).to(torch.bfloat16).float().numpy()
        np.testing.assert_array_equal(kb, want)
        r = ob["r"]
        req1 = alpa.InferenceRequest(num_trajectories=4, v0=5.0, topology="multi")
        g.set_lane_prefix(np.array([0, 1, 2, 1], np.int32))
        in_place = g.run_action_generation(req1)
        # compact copy [lanes][B][2][r][kv] of the same bf16 values, bound from the host
        g.bind_prefix(np.ascontiguousarray(kb))
        compact = g.run_action_generation(req1)
        np.testing.assert_array_equal(in_place.actions, compact.actions)
        g.set_lane_prefix(np.zeros(0, np.int32))
        # single topology: one reasoning lane shared by every trajectory
        o1 = g.run_reasoning(vis, prompt, lanes=1, max_new_tokens=40, sampler_seed=5)
        k1 = device_prefix(g, 1, 2, cap, 128, o1["r"], dtype="bf16")
        req = alpa.InferenceRequest(num_trajectories=6, v0=5.0)
        in_place = g.run_action_generation(req)
        g.bind_prefix(np.ascontiguousarray(k1[0]))
        compact = g.run_action_generation(req)
        np.testing.assert_array_equal(in_place.actions, compact.actions)
    assert r == ob["r"]
