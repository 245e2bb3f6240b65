"""GPU parity: the sm_100a path through the C-ABI vs the CPU oracle.

Bars (BASELINE.json north_star):
  * fp32 path:  rel-L2 <= 1e-4 on actions and trajectories (config 1),
  * bf16 path:  rel-L2 <= 2e-2 (config-2 width, reduced B / K so the oracle
    finishes in seconds),
  * rollout / indexing / seeding: bit-exact.
Reference known-answer tests restated on the device path:
test_model.cpp:288-447, test_pipeline.cpp:247-349.
"""
import numpy as np
import pytest

import paper_2605_08975_b200 as alpa
from oracle.oracle import Cfg

pytestmark = pytest.mark.gpu

F32_TOL = 1e-4
BF16_TOL = 2e-2


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def c1(**kw):
    return alpa.ModelConfig(**kw)


def ocfg(m: alpa.ModelConfig) -> Cfg:
    return Cfg.make(vision_blocks=m.vision_blocks, decoder_blocks=m.decoder_blocks,
                    hidden_dim=m.hidden_dim, action_hidden_dim=m.action_hidden_dim,
                    kv_dim=m.kv_dim, heads=m.heads, vocab_size=m.vocab_size,
                    patch_size=m.patch_size, diffusion_iters=m.diffusion_iters,
                    update_scale=m.update_scale, weight_seed=m.weight_seed)


@pytest.fixture(scope="module")
def gen_c1(golden):
    g = alpa.ActionGenerator(c1())
    g.bind_prefix(golden["prefix"])
    yield g
    g.close()


# ----------------------------------------------------------------- config 1 (fp32)
@pytest.mark.parametrize("n,k", [(1, 10), (6, 10), (16, 10), (6, 1), (6, 5)])
def test_config1_f32_parity(gen_c1, golden, n, k):
    req = alpa.InferenceRequest(num_trajectories=n, diffusion_iters=k, v0=golden["v0"])
    res = gen_c1.run_action_generation(req)
    ea = golden["expected"][f"n{n}_k{k}_actions"]
    et = golden["expected"][f"n{n}_k{k}_traj"]
    assert rel_l2(res.actions, ea) <= F32_TOL
    assert rel_l2(res.trajectories, et) <= F32_TOL
    assert res.stats["graph_launches"] == 1
    assert res.stats["kernel_launches"] > 0


def test_config1_rollout_of_gpu_actions_is_bitexact(gen_c1, golden, port):
    req = alpa.InferenceRequest(num_trajectories=6, v0=golden["v0"])
    res = gen_c1.run_action_generation(req)
    np.testing.assert_array_equal(res.trajectories, port.rollout(res.actions, golden["v0"]))


def test_graph_equals_eager_bitwise(gen_c1, golden):
    # test_model.cpp:357-377 / acceptance.cpp:92-127
    base = dict(num_trajectories=6, v0=golden["v0"])
    g = gen_c1.run_action_generation(alpa.InferenceRequest(executor="graph", **base))
    e = gen_c1.run_action_generation(alpa.InferenceRequest(executor="eager", **base))
    d = gen_c1.run_action_generation(alpa.InferenceRequest(executor="eager",
                                                           kv_strategy="dynamic", **base))
    np.testing.assert_array_equal(g.actions, e.actions)
    np.testing.assert_array_equal(g.trajectories, d.trajectories)
    assert e.stats["graph_launches"] == 0


def test_repeat_calls_deterministic(gen_c1, golden):
    req = alpa.InferenceRequest(num_trajectories=6, v0=golden["v0"])
    a = gen_c1.run_action_generation(req)
    b = gen_c1.run_action_generation(req)
    np.testing.assert_array_equal(a.actions, b.actions)


def test_stride_zero_identical_lanes(gen_c1, golden):
    # test_pipeline.cpp:247-273
    res = gen_c1.run_action_generation(alpa.InferenceRequest(num_trajectories=3,
                                                             action_seed_stride=0,
                                                             v0=golden["v0"]))
    np.testing.assert_array_equal(res.actions[0], res.actions[1])
    np.testing.assert_array_equal(res.trajectories[0], res.trajectories[2])
    res = gen_c1.run_action_generation(alpa.InferenceRequest(num_trajectories=2, v0=5.0))
    assert np.abs(res.actions[0] - res.actions[1]).max() > 0


def test_lane_slices_keep_global_seeds(gen_c1, golden):
    # multi-GPU slicing: lanes [2,6) computed alone equal
    # lanes 2..5 of the full N=6 run.
    full = gen_c1.run_action_generation(alpa.InferenceRequest(num_trajectories=6, v0=5.0))
    part = gen_c1.run_action_generation(alpa.InferenceRequest(num_trajectories=4, lane0=2,
                                                              v0=5.0))
    np.testing.assert_array_equal(full.actions[2:], part.actions)


def test_lane_permutation_bitwise(port):
    # test_model.cpp:426-447, through the device path: permute the per-lane
    # noise seeds (stride trick) and compare lanes.
    cfg = alpa.ModelConfig(vision_blocks=1, decoder_blocks=2, hidden_dim=16, action_hidden_dim=8,
                           kv_dim=8, heads=2, vocab_size=128, weight_seed=77)
    with alpa.ActionGenerator(cfg) as g:
        g.bind_prefix(port.synthetic_prefix(55, 2, 10, 8))
        fwd = g.run_action_generation(alpa.InferenceRequest(num_trajectories=2, action_init_seed=1,
                                                            action_seed_stride=1, v0=1.0))
        rev = g.run_action_generation(alpa.InferenceRequest(num_trajectories=2, action_init_seed=2,
                                                            action_seed_stride=2**64 - 1, v0=1.0))
        np.testing.assert_array_equal(fwd.actions[0], rev.actions[1])
        np.testing.assert_array_equal(fwd.actions[1], rev.actions[0])


def test_zero_head_identity_and_unit_delta(port):
    # test_model.cpp:322-355 through alpa_load_weights_host
    cfg = alpa.ModelConfig(vision_blocks=1, decoder_blocks=2, hidden_dim=16, action_hidden_dim=8,
                           kv_dim=8, heads=2, vocab_size=128, weight_seed=77, diffusion_iters=1)
    w = port.weights(ocfg(cfg))
    arena = w.arena().copy()
    hw, hb = w.tensor("head")
    nh = hw.size + hb.size
    arena[-nh:] = 0.0
    pre = port.synthetic_prefix(4, 2, 10, 8)
    with alpa.ActionGenerator(cfg, weights=arena) as g:
        g.bind_prefix(pre)
        res = g.run_action_generation(alpa.InferenceRequest(num_trajectories=1,
                                                            action_init_seed=9,
                                                            action_seed_stride=0, v0=1.0))
        np.testing.assert_array_equal(res.actions, alpa.host_noise(9, 0, 1))
    arena[-hb.size:] = 1.0
    cfg10 = alpa.ModelConfig(**{**cfg.__dict__, "diffusion_iters": 10})
    with alpa.ActionGenerator(cfg10, weights=arena) as g:
        g.bind_prefix(pre)
        res = g.run_action_generation(alpa.InferenceRequest(num_trajectories=1, v0=1.0))
        # every step adds 0.1 * 1.0: the noise init moves by K * 0.1 = 1.0
        np.testing.assert_allclose(res.actions - alpa.host_noise(2, 1, 1), 1.0, atol=1e-5)


def test_device_weights_match_host_arena(port):
    # on-device splitmix jump-ahead == host arena upload (bitwise end to end)
    cfg = alpa.ModelConfig(vision_blocks=1, decoder_blocks=2, hidden_dim=16, action_hidden_dim=8,
                           kv_dim=8, heads=2, vocab_size=128, weight_seed=77)
    arena = port.weights(ocfg(cfg)).arena().copy()
    pre = port.synthetic_prefix(4, 2, 12, 8)
    req = alpa.InferenceRequest(num_trajectories=2, v0=2.0)
    with alpa.ActionGenerator(cfg) as g1, alpa.ActionGenerator(cfg, weights=arena) as g2:
        g1.bind_prefix(pre)
        g2.bind_prefix(pre)
        np.testing.assert_array_equal(g1.run_action_generation(req).actions,
                                      g2.run_action_generation(req).actions)


def test_synthetic_prefix_on_device_matches_host(port):
    cfg = alpa.ModelConfig(vision_blocks=1, decoder_blocks=2, hidden_dim=16, action_hidden_dim=8,
                           kv_dim=8, heads=2, vocab_size=128, weight_seed=77)
    req = alpa.InferenceRequest(num_trajectories=2, v0=2.0)
    with alpa.ActionGenerator(cfg) as g:
        g.bind_prefix(port.synthetic_prefix(4242, 2, 33, 8))
        a = g.run_action_generation(req).actions
        g.bind_prefix_synthetic(4242, 33)
        b = g.run_action_generation(req).actions
    np.testing.assert_array_equal(a, b)


def test_multi_topology_matches_oracle(port):
    m = alpa.ModelConfig(vision_blocks=2, decoder_blocks=3, hidden_dim=32, action_hidden_dim=16,
                         kv_dim=16, heads=4, vocab_size=256, weight_seed=9001)
    n, r = 3, 20
    pre = np.stack([port.synthetic_prefix(88 + 100 * l, 3, r, 16) for l in range(n)])
    exp = port.refine(ocfg(m), port.weights(ocfg(m)), pre, port.noise(2, 1, n),
                      lane_prefix=np.arange(n, dtype=np.int32))
    with alpa.ActionGenerator(m) as g:
        g.bind_prefix(pre)
        res = g.run_action_generation(alpa.InferenceRequest(num_trajectories=n, topology="multi",
                                                            v0=1.0))
    assert rel_l2(res.actions, exp) <= F32_TOL


# ----------------------------------------------------------------- rollout
def test_device_rollout_bitexact_random(port):
    rng = np.random.default_rng(1234)
    n = 20000
    acts = (rng.standard_normal((n, 64, 2)) * np.array([2.0, 0.3])).astype(np.float32)
    with alpa.ActionGenerator(c1()) as g:
        for v0 in (0.0, 5.0, 17.3):
            got = g.rollout(acts, v0)
            exp = port.rollout(acts, v0)
            mism = int(np.sum(got.view(np.uint32) != exp.view(np.uint32)))
            assert mism == 0, f"{mism} mismatching floats at v0={v0}"


def test_rollout_known_answers():
    with alpa.ActionGenerator(c1()) as g:
        a = np.zeros((1, 64, 2), np.float32)
        t = g.rollout(a, 1.0)[0]
        np.testing.assert_allclose(t[:, 0], 0.1 * np.arange(1, 65), rtol=1e-6)
        a[0, 3, 0] = np.nan
        with pytest.raises(alpa.InternalError):
            g.rollout(a, 1.0)
        with pytest.raises(alpa.InternalError):
            g.rollout(np.zeros((1, 64, 2), np.float32), -1.0)


# ----------------------------------------------------------------- errors
def test_error_taxonomy(gen_c1, golden):
    with pytest.raises(alpa.ConfigError):
        gen_c1.run_action_generation(alpa.InferenceRequest(num_trajectories=0))
    with pytest.raises(alpa.ConfigError):  # model.cpp:609-611
        gen_c1.run_action_generation(alpa.InferenceRequest(num_trajectories=1, executor="graph",
                                                           kv_strategy="dynamic"))
    with alpa.ActionGenerator(c1()) as g:
        with pytest.raises(alpa.InternalError):  # unsealed / missing prefix
            g.run_action_generation(alpa.InferenceRequest(num_trajectories=1))
        g.bind_prefix(np.stack([golden["prefix"]] * 2))
        with pytest.raises(alpa.InternalError):  # single topology needs batch-1 source
            g.run_action_generation(alpa.InferenceRequest(num_trajectories=2, topology="single"))
        with pytest.raises(alpa.InternalError):  # kv batch != N (pipeline.cpp:411-413)
            g.run_action_generation(alpa.InferenceRequest(num_trajectories=3, topology="multi"))


# ----------------------------------------------------------------- bf16 tensor-core path
def c2(B=2, K=2, **kw):
    d = dict(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=B,
             action_hidden_dim=2048, kv_dim=1024, heads=8, diffusion_iters=K, dtype="bf16")
    d.update(kw)
    return alpa.ModelConfig(**d)


@pytest.mark.parametrize("n,B,K,r", [(6, 2, 2, 512), (1, 1, 1, 256), (16, 1, 1, 128)])
def test_bf16_config2_width_parity(port, n, B, K, r):
    m = c2(B=B, K=K)
    pre = port.synthetic_prefix(4242, B, r, m.kv_dim)
    exp = port.refine(ocfg(m), port.weights(ocfg(m)), pre, port.noise(2, 1, n))
    with alpa.ActionGenerator(m) as g:
        g.bind_prefix_synthetic(4242, r)
        res = g.run_action_generation(alpa.InferenceRequest(num_trajectories=n, v0=5.0))
    err = rel_l2(res.actions, exp)
    print(f"bf16 n={n} B={B} K={K} r={r}: rel-L2 {err:.3e}")
    assert err <= BF16_TOL
    assert rel_l2(res.trajectories, port.rollout(exp, 5.0)) <= BF16_TOL


def test_bf16_small_width(port):
    m = c2(B=2, K=3, action_hidden_dim=256, kv_dim=128, heads=2)
    pre = port.synthetic_prefix(7, 2, 100, 128)
    exp = port.refine(ocfg(m), port.weights(ocfg(m)), pre, port.noise(2, 1, 6))
    with alpa.ActionGenerator(m) as g:
        g.bind_prefix(pre)
        res = g.run_action_generation(alpa.InferenceRequest(num_trajectories=6, v0=5.0))
        res2 = g.run_action_generation(alpa.InferenceRequest(num_trajectories=6, v0=5.0,
                                                             executor="eager"))
    err = rel_l2(res.actions, exp)
    print(f"bf16 small width rel-L2 {err:.3e}")
    assert err <= BF16_TOL
    np.testing.assert_array_equal(res.actions, res2.actions)  # deterministic split-K


@pytest.mark.parametrize("r,splits", [(1000, "1"), (256, "2"), (2048, None)])
def test_bf16_attention_kv_splits(port, monkeypatch, r, splits):
    # multi-block online softmax (rescale of the TMEM accumulator) and the
    # cluster/DSMEM split combine, incl. a prefix length that is not a
    # multiple of the 128-key block.
    if splits:
        monkeypatch.setenv("ALPA_ATTN_SPLITS", splits)
    B = 1
    m = c2(B=B, K=1) if r == 2048 else c2(B=B, K=1, action_hidden_dim=256, kv_dim=128, heads=1)
    pre = port.synthetic_prefix(7, B, r, m.kv_dim)
    exp = port.refine(ocfg(m), port.weights(ocfg(m)), pre, port.noise(2, 1, 6))
    with alpa.ActionGenerator(m) as g:
        g.bind_prefix(pre)
        res = g.run_action_generation(alpa.InferenceRequest(num_trajectories=6, v0=5.0))
    err = rel_l2(res.actions, exp)
    print(f"bf16 attention r={r} splits={splits}: rel-L2 {err:.3e}")
    assert err <= BF16_TOL


# ----------------------------------------------------------------- persistent kernel
@pytest.mark.parametrize("n,B,K,r", [(6, 2, 2, 300), (3, 1, 1, 700), (5, 1, 2, 200), (11, 1, 1, 130)])
def test_persistent_kernel_vs_per_op_path(port, monkeypatch, n, B, K, r):
    """The persistent iteration kernel (default) and the per-op kernel sequence
    (ALPA_MK=0) compute the same iteration: both within the bf16 bar of the
    oracle, and each deterministic (graph replay == eager launch, bitwise).
    Covers an odd lane count (partial 128-row query tile, half token tiles)
    and a prefix that is not a multiple of the 64-key block."""
    m = c2(B=B, K=K)
    pre = port.synthetic_prefix(4242, B, r, m.kv_dim)
    exp = port.refine(ocfg(m), port.weights(ocfg(m)), pre, port.noise(2, 1, n))
    out = {}
    for mk in ("1", "0"):
        monkeypatch.setenv("ALPA_MK", mk)
        with alpa.ActionGenerator(m) as g:
            g.bind_prefix_synthetic(4242, r)
            res = g.run_action_generation(alpa.InferenceRequest(num_trajectories=n, v0=5.0))
            res_e = g.run_action_generation(alpa.InferenceRequest(num_trajectories=n, v0=5.0,
                                                                  executor="eager"))
        np.testing.assert_array_equal(res.actions, res_e.actions)
        out[mk] = res.actions
        err = rel_l2(res.actions, exp)
        print(f"ALPA_MK={mk} n={n} B={B} K={K} r={r}: rel-L2 {err:.3e}")
        assert err <= BF16_TOL
    assert rel_l2(out["1"], out["0"]) <= BF16_TOL


@pytest.mark.parametrize("n,B,K,r,lane_map", [(3, 2, 2, 300, None), (5, 1, 2, 130, [2, 0, 2, 1, 0])])
def test_persistent_kernel_multi_topology(port, monkeypatch, n, B, K, r, lane_map):
    """Multi topology (lane l attends prefix lane_map[l], pipeline.cpp:405-413)
    on the persistent kernel: one query tile per lane, the lane's prefix rows
    read from the device lane map.  Within the bf16 bar of the oracle, equal
    to the per-op path within the bar, graph == eager bitwise, and one
    persistent launch per iteration (the persistent kernel really ran)."""
    m = c2(B=B, K=K)
    npre = 3 if lane_map else n
    pre = np.stack([port.synthetic_prefix(500 + 100 * l, B, r, m.kv_dim) for l in range(npre)])
    lp = np.array(lane_map if lane_map else list(range(n)), np.int32)
    exp = port.refine(ocfg(m), port.weights(ocfg(m)), pre, port.noise(2, 1, n), lane_prefix=lp)
    out = {}
    for mk in ("1", "0"):
        monkeypatch.setenv("ALPA_MK", mk)
        with alpa.ActionGenerator(m) as g:
            g.bind_prefix(pre)
            if lane_map:
                g.set_lane_prefix(lp)
            req = alpa.InferenceRequest(num_trajectories=n, topology="multi", v0=5.0)
            res = g.run_action_generation(req)
            res_e = g.run_action_generation(alpa.InferenceRequest(num_trajectories=n, topology="multi",
                                                                  v0=5.0, executor="eager"))
        np.testing.assert_array_equal(res.actions, res_e.actions)
        if mk == "1":
            assert res.stats["kernel_launches"] == K + 1
        out[mk] = res.actions
        err = rel_l2(res.actions, exp)
        print(f"multi ALPA_MK={mk} n={n} B={B} K={K} r={r} map={lp.tolist()}: rel-L2 {err:.3e}")
        assert err <= BF16_TOL
    assert rel_l2(out["1"], out["0"]) <= BF16_TOL


@pytest.mark.parametrize("topology", ["single", "multi"])
def test_bf16_compare_actiongen_variants(port, topology):
    """cmd_compare_actiongen (cli.cpp:236-313) on the bf16 tensor-core path:
    the reference's three variants (baseline = dynamic KV + eager, +static_kv,
    +graph) produce bitwise-equal actions (cli.cpp:292-300), for the shared
    prefix and for per-lane prefixes; graph + dynamic is a ConfigError
    (model.cpp:609-611)."""
    m = c2(B=2, K=2)
    n, r = 4, 200
    if topology == "single":
        pre = port.synthetic_prefix(4242, 2, r, m.kv_dim)
    else:
        pre = np.stack([port.synthetic_prefix(900 + l, 2, r, m.kv_dim) for l in range(n)])
    variants = {"baseline": ("dynamic", "eager"), "+static_kv": ("static", "eager"),
                "+graph": ("static", "graph")}
    got = {}
    with alpa.ActionGenerator(m) as g:
        g.bind_prefix(pre)
        for name, (kv, ex) in variants.items():
            res = g.run_action_generation(alpa.InferenceRequest(
                num_trajectories=n, topology=topology, kv_strategy=kv, executor=ex, v0=5.0))
            got[name] = res
        with pytest.raises(alpa.ConfigError):
            g.run_action_generation(alpa.InferenceRequest(num_trajectories=n, topology=topology,
                                                          kv_strategy="dynamic", executor="graph"))
    for name in variants:
        np.testing.assert_array_equal(got[name].actions, got["baseline"].actions)
        np.testing.assert_array_equal(got[name].trajectories, got["baseline"].trajectories)
    lp = None if topology == "single" else np.arange(n, dtype=np.int32)
    exp = port.refine(ocfg(m), port.weights(ocfg(m)), pre, port.noise(2, 1, n), lane_prefix=lp)
    assert rel_l2(got["baseline"].actions, exp) <= BF16_TOL


def test_persistent_kernel_single_launch_per_iteration(port):
    """One persistent launch per denoising iteration (+ the rollout)."""
    m = c2(B=2, K=3, action_hidden_dim=256, kv_dim=128, heads=1)
    with alpa.ActionGenerator(m) as g:
        g.bind_prefix(port.synthetic_prefix(7, 2, 100, 128))
        res = g.run_action_generation(alpa.InferenceRequest(num_trajectories=6, v0=5.0))
    assert res.stats["kernel_launches"] == 3 + 1


# ----------------------------------------------------------------- open-loop metrics
@pytest.mark.parametrize("scenes,n", [(1, 2), (3, 6), (2, 16), (5, 1)])
def test_device_open_loop_metrics_bitexact(port, scenes, n):
    """Device min_ade / diversity of a scene batch == the reference's
    (eval.cpp:39-59) bitwise, on random trajectories and on generated ones."""
    from oracle.oracle import Ref, have_ref
    oracle = Ref() if have_ref() else port
    rng = np.random.default_rng(scenes * 100 + n)
    t = (rng.standard_normal((scenes, n, 64, 3)) * 10).astype(np.float32)
    g = (rng.standard_normal((scenes, 64, 3)) * 10).astype(np.float32)
    with alpa.ActionGenerator(c1()) as gen:
        ade, div = gen.eval_open_loop(t, g, diversity=n > 1)
        for s in range(scenes):
            assert ade[s] == oracle.min_ade(t[s], g[s])
            if n > 1:
                assert div[s] == oracle.diversity(t[s])
        if n == 1:
            with pytest.raises(alpa.InternalError):
                gen.eval_open_loop(t, g, diversity=True)


def test_device_open_loop_metrics_on_generated(gen_c1, golden, port):
    res = gen_c1.run_action_generation(alpa.InferenceRequest(num_trajectories=6, v0=golden["v0"]))
    gt = res.trajectories[0] * 0.5
    ade, div = gen_c1.eval_open_loop(res.trajectories, gt)
    assert ade[0] == port.min_ade(res.trajectories, gt)
    assert div[0] == port.diversity(res.trajectories)


# ----------------------------------------------------------------- shape sweep (edge cases)
@pytest.mark.parametrize("n,r,topology", [
    (1, 1, "single"), (2, 63, "single"), (3, 64, "multi"), (5, 65, "single"), (7, 127, "multi"),
    (9, 129, "single"), (13, 300, "multi"), (17, 777, "single"), (20, 2048, "single"),
])
def test_persistent_kernel_shape_sweep(port, n, r, topology):
    """The persistent tensor-core kernel over ragged shapes vs the oracle (bf16
    bar): prefix lengths around the 64-key block (1, 63-65, 127-129), odd and
    large lane counts (partial query tiles, several items per CTA), single and
    multi topology; graph == eager bitwise for each."""
    m = c2(B=1, K=1)
    if topology == "single":
        pre = port.synthetic_prefix(31 + r, 1, r, m.kv_dim)
        lp = None
    else:
        pre = np.stack([port.synthetic_prefix(71 + l, 1, r, m.kv_dim) for l in range(n)])
        lp = np.arange(n, dtype=np.int32)
    exp = port.refine(ocfg(m), port.weights(ocfg(m)), pre, port.noise(2, 1, n), lane_prefix=lp)
    with alpa.ActionGenerator(m) as g:
        g.bind_prefix(pre)
        res = g.run_action_generation(alpa.InferenceRequest(num_trajectories=n, topology=topology, v0=5.0))
        res_e = g.run_action_generation(alpa.InferenceRequest(num_trajectories=n, topology=topology, v0=5.0,
                                                              executor="eager"))
    np.testing.assert_array_equal(res.actions, res_e.actions)
    err = rel_l2(res.actions, exp)
    print(f"sweep n={n} r={r} {topology}: rel-L2 {err:.3e}")
    assert err <= BF16_TOL
    assert res.stats["kernel_launches"] == 1 + 1
