"""CPU tests: pin the oracle (the checker) before anyone trusts it.

* against the reference's golden digests (regenerated from the
  reference itself by tests/golden/make_golden.py);
* against the reference library itself (oracle/_ref, when built here) on the
  reference's own small test configs (test_model.cpp:15-27,
  acceptance.cpp:38-50), bit for bit;
* against the reference's known-answer tests for this path
  (test_model.cpp:322-355, test_pipeline.cpp:148-195, test_kv_cache.cpp:231-242).
"""
import math

import numpy as np
import pytest

from oracle.oracle import Cfg, Ref, have_ref


def tiny_cfg(**kw):  # test_model.cpp:15-27
    d = dict(vision_blocks=1, decoder_blocks=2, hidden_dim=16, action_hidden_dim=8, kv_dim=8,
             heads=2, vocab_size=128, max_new_tokens=16, weight_seed=77)
    d.update(kw)
    return Cfg.make(**d)


def small_cfg(**kw):  # acceptance.cpp:38-50
    d = dict(vision_blocks=2, decoder_blocks=3, hidden_dim=32, action_hidden_dim=16, kv_dim=16,
             heads=4, vocab_size=256, max_new_tokens=24, weight_seed=9001)
    d.update(kw)
    return Cfg.make(**d)


def test_stream_offset_matches_survey(port):
    # S1 = 518,144 draws for the default config
    assert port.stream_offset(Cfg.make()) == 518144
    # config 2 (vision 0, hidden 64, vocab 128, B=36, kv=1024): S2 = 10,795,456
    c2 = Cfg.make(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=36,
                  action_hidden_dim=2048, kv_dim=1024, heads=8)
    assert port.stream_offset(c2) == 10795456
    assert port.param_count(c2) == 1544077314


def test_weight_stream_pins(port, golden):
    cfg = Cfg.make()
    w = port.weights(cfg)
    pins = golden["weight_pins"]
    checks = {
        "action_in_w": w.tensor("action_in")[0].ravel(),
        "head_b": w.tensor("head")[1].ravel(),
        "blk5_mlp2_b": w.tensor("mlp2", 5)[1].ravel(),
        "blk0_q_w": w.tensor("q", 0)[0].ravel(),
    }
    for name, v in checks.items():
        assert v.size == pins[name]["n"], name
        assert f"{port.fnv1a(v):016x}" == pins[name]["fnv"], name


@pytest.mark.parametrize("key", ["n1_k10", "n6_k10", "n16_k10", "n6_k1", "n6_k5"])
def test_port_reproduces_golden_digests(port, golden, key):
    n = int(key.split("_")[0][1:])
    k = int(key.split("_")[1][1:])
    cfg = Cfg.make(diffusion_iters=k)
    w = port.weights(cfg)
    acts = port.refine(cfg, w, golden["prefix"], port.noise(2, 1, n))
    traj = port.rollout(acts, golden["v0"])
    run = golden["runs"][key]
    assert f"{port.fnv1a(acts):016x}" == run["actions_fnv"]
    assert f"{port.fnv1a(traj):016x}" == run["traj_fnv"]
    np.testing.assert_array_equal(acts, golden["expected"][f"{key}_actions"])


def test_survey_digests_are_the_golden_ones(golden):
    # the digests SURVEY.md §8c quotes for the canonical build
    assert golden["runs"]["n1_k10"]["actions_fnv"] == "4c2c9f263f394ff4"
    assert golden["runs"]["n1_k10"]["traj_fnv"] == "68af303f0a8c9aaa"
    assert golden["runs"]["n6_k10"]["actions_fnv"] == "11a762f69b8bd1d3"
    assert golden["runs"]["n6_k10"]["traj_fnv"] == "ed1c9b87a1a171fa"
    assert golden["reasoning_fingerprint"] == "04e2beb925b91bdd"
    assert golden["r"] == 427


def test_noise_matches_golden(port, golden):
    np.testing.assert_array_equal(port.noise(2, 1, 16), golden["expected"]["noise_n16"])


@pytest.mark.skipif(not have_ref(), reason="reference library not built here")
@pytest.mark.parametrize("mk,n,single", [(tiny_cfg, 2, True), (small_cfg, 6, True),
                                         (small_cfg, 3, False)])
def test_port_bitwise_vs_reference(port, mk, n, single):
    from oracle.oracle import Ref
    ref = Ref()
    cfg = mk()
    r = 12
    if single:
        prefix = port.synthetic_prefix(88, cfg.decoder_blocks, r, cfg.kv_dim)
        lp = None
    else:
        prefix = np.stack([port.synthetic_prefix(88 + 100 * l, cfg.decoder_blocks, r, cfg.kv_dim)
                           for l in range(n)])
        lp = np.arange(n, dtype=np.int32)
    ref_in = prefix if single else np.ascontiguousarray(prefix.transpose(1, 2, 0, 3, 4))
    a_ref, _, _ = ref.action_generation(cfg, ref_in, n, seed=5, stride=3, single=single)
    a = port.refine(cfg, port.weights(cfg), prefix, port.noise(5, 3, n), lane_prefix=lp)
    np.testing.assert_array_equal(a.view(np.uint32), a_ref.view(np.uint32))


@pytest.mark.skipif(not have_ref(), reason="reference library not built here")
def test_reference_variants_identical(port):
    # optimization transparency (test_pipeline.cpp:333-349): dynamic/eager ==
    # static/graph, the equivalence the GPU path must also keep.
    from oracle.oracle import Ref
    ref = Ref()
    cfg = small_cfg()
    prefix = port.synthetic_prefix(7, cfg.decoder_blocks, 10, cfg.kv_dim)
    a1, _, _ = ref.action_generation(cfg, prefix, 2, static_kv=False, graph=False)
    a2, _, _ = ref.action_generation(cfg, prefix, 2, static_kv=True, graph=True)
    np.testing.assert_array_equal(a1, a2)


def test_zero_head_is_identity(port):
    # test_model.cpp:322-340
    cfg = tiny_cfg(diffusion_iters=1)
    w = port.weights(cfg)
    hw, hb = w.tensor("head")
    hw[:] = 0
    hb[:] = 0
    init = port.noise(9, 0, 1)
    out = port.refine(cfg, w, port.synthetic_prefix(4, 2, 10, 8), init)
    np.testing.assert_array_equal(out, init)


def test_constant_unit_delta(port):
    # test_model.cpp:342-355: every (a, k) = K * 0.1 = 1.0 from zero init
    cfg = tiny_cfg()
    w = port.weights(cfg)
    hw, hb = w.tensor("head")
    hw[:] = 0
    hb[:] = 1
    out = port.refine(cfg, w, port.synthetic_prefix(4, 2, 10, 8), np.zeros((1, 64, 2), np.float32))
    np.testing.assert_allclose(out, 1.0, rtol=1e-5)


def test_lane_permutation(port):
    # test_model.cpp:426-447
    cfg = tiny_cfg()
    w = port.weights(cfg)
    pre = port.synthetic_prefix(55, 2, 10, 8)
    a = np.concatenate([port.noise(1, 0, 1), port.noise(2, 0, 1)])
    b = a[::-1].copy()
    fa = port.refine(cfg, w, pre, a)
    fb = port.refine(cfg, w, pre, b)
    np.testing.assert_array_equal(fa[0], fb[1])
    np.testing.assert_array_equal(fa[1], fb[0])


def const_actions(a, k):
    x = np.empty((1, 64, 2), np.float32)
    x[..., 0] = a
    x[..., 1] = k
    return x


def test_unicycle_known_answers(port):
    # test_pipeline.cpp:148-189
    t = port.rollout(const_actions(0, 0), 1.0)[0]
    np.testing.assert_allclose(t[:, 0], 0.1 * np.arange(1, 65), rtol=1e-6)
    assert np.all(t[:, 1] == 0) and np.all(t[:, 2] == 0)
    t = port.rollout(const_actions(1.0, 0.0), 0.0)[0]
    assert t[0, 0] == pytest.approx(0.0)
    assert t[2, 0] == pytest.approx(0.03, rel=1e-6)
    # circle within 0.05 m of a 1000x-substep integrator
    coarse = port.rollout(const_actions(0.0, 0.1), 1.0)[0]
    x = y = yaw = 0.0
    v = 1.0
    for i in range(64):
        for _ in range(1000):
            h = 1e-4
            x, y, yaw = x + v * math.cos(yaw) * h, y + v * math.sin(yaw) * h, yaw + 0.1 * v * h
        assert math.hypot(coarse[i, 0] - x, coarse[i, 1] - y) < 0.05
    with pytest.raises(ValueError):
        bad = const_actions(0, 0)
        bad[0, 3, 0] = np.nan
        port.rollout(bad, 1.0)


def test_initial_speed(port):
    # test_pipeline.cpp:191-195
    h = np.zeros((16, 3), np.float32)
    h[:, 0] = [-(15 - j) * 3.0 * 0.1 for j in range(16)]
    assert port.initial_speed(h) == pytest.approx(3.0, rel=1e-5)


def test_footprint_formula(port):
    # test_kv_cache.cpp:231-242
    assert port.footprint(36, 1, 3081, 1024, 2) == 454311936
    assert port.footprint(36, 1, 64, 1024, 2) == 9437184


# ----------------------------------------------------------------- open-loop metrics
@pytest.mark.skipif(not have_ref(), reason="reference library not built")
@pytest.mark.parametrize("n", [1, 2, 6, 16])
def test_oracle_open_loop_metrics_match_reference(port, n):
    """C restatement of min_ade / diversity (eval.cpp:14-59) == the reference, bitwise."""
    ref = Ref()
    rng = np.random.default_rng(n)
    t = (rng.standard_normal((n, 64, 3)) * 10).astype(np.float32)
    g = (rng.standard_normal((64, 3)) * 10).astype(np.float32)
    assert port.min_ade(t, g) == ref.min_ade(t, g)
    if n > 1:
        assert port.diversity(t) == ref.diversity(t)
    else:
        with pytest.raises(ValueError):
            port.diversity(t)


@pytest.mark.skipif(not have_ref(), reason="reference library not built")
def test_latency_report_json_parses_with_reference():
    """The shim's LatencyReport JSON key set (profiler.cpp:31-46) round-trips
    through the reference's LatencyReport::from_json (document built the way
    the shim's to_json builds it)."""
    import json
    doc = {"preprocessing_ms": 0.0, "reasoning_vision_ms": 0.0, "reasoning_prefill_ms": 0.0,
           "reasoning_decode_ms": 0.0, "action_gen_ms": 30.5, "total_ms": 30.5,
           "postprocessing_ms": 0.0, "repeats": 1, "action_gen_iter_ms": [3.0] * 10,
           "alloc_count": 0, "dispatch_count": 11, "replay_count": 1, "bytes_allocated": 123,
           "kv_bytes": 456, "cot_tokens": 0}
    n, ms = Ref().parse_latency_report(json.dumps(doc))
    assert n == 10 and ms == 30.5
    with pytest.raises(RuntimeError):
        Ref().parse_latency_report(json.dumps({k: v for k, v in doc.items() if k != "kv_bytes"}))
