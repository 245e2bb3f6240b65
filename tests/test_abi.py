"""CPU tests of the drop-in boundary (no compute calls without a GPU).

* libalpa_action.so loads and exports every symbol include/alpa_action.h
  declares;
* the host-side helpers are bit-exact restatements of the reference host code
  (noise, initial speed, footprint, weight-stream offset, config validation);
* without a GPU the library refuses to run (no CPU fallback).
"""
import os
import re

import numpy as np
import pytest

import paper_2605_08975_b200 as alpa
from oracle.oracle import Cfg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "alpa_action.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(alpa_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = alpa.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), f"{s} missing from libalpa_action.so"


def test_library_contains_tcgen05_and_tma_sass():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", alpa.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "UTCHMMA" in out      # tcgen05.mma
    assert "UTMALDG" in out      # TMA loads
    assert "LDTM" in out         # tcgen05.ld (TMEM -> registers)


def test_host_noise_bitexact(port):
    for seed, stride, lane0, n in [(2, 1, 0, 6), (123456789, 7, 3, 4), (0, 0, 0, 2)]:
        a = alpa.host_noise(seed, stride, n, lane0)
        b = port.noise(seed, stride, n, lane0)
        np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))


def test_initial_speed_matches_oracle(port):
    rng = np.random.default_rng(0)
    for _ in range(20):
        h = rng.normal(size=(16, 3)).astype(np.float32)
        assert alpa.initial_speed(h) == port.initial_speed(h)


def test_footprint_and_offsets(port):
    assert alpa.kv_footprint_bytes(36, 1, 3081, 1024, 2) == 454311936
    cfg = alpa.ModelConfig()
    assert cfg.weight_stream_offset() == port.stream_offset(Cfg.make()) == 518144
    c2 = alpa.ModelConfig(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=36,
                          action_hidden_dim=2048, kv_dim=1024, heads=8, dtype="bf16")
    assert c2.weight_stream_offset() == 10795456
    assert c2.action_param_count() == 1544077314


@pytest.mark.parametrize("bad", [dict(kv_dim=7), dict(update_scale=0.0), dict(action_steps=32),
                                 dict(decoder_blocks=0), dict(diffusion_iters=0),
                                 dict(dtype="bf16")])
def test_config_validation_is_configerror(bad):
    # test_model.cpp:78-89 (+ the bf16 tile constraint of this build)
    cfg = alpa.ModelConfig(**bad)
    with pytest.raises(alpa.ConfigError):
        cfg.validate()


def test_default_config_valid():
    alpa.ModelConfig().validate()
    alpa.ModelConfig(action_hidden_dim=2048, kv_dim=1024, heads=8, dtype="bf16").validate()


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(alpa.InternalError, match="no CUDA device"):
        alpa.ActionGenerator(alpa.ModelConfig())


def test_host_sampler_matches_restatement():
    """alpa_sample_token (host, no GPU): sample_token (model.cpp:30-54) --
    greedy argmax, and the temperature-1 CDF walk in double over
    Rng::next_float (splitmix64 >> 40, common.hpp:36-59)."""
    import math

    def splitmix(state):
        state = (state + 0x9E3779B97F4A7C15) & (2**64 - 1)
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        return state, z ^ (z >> 31)

    def ref_sample(lg, state):
        mx = max(float(v) for v in lg)
        tot = sum(math.exp(float(v) - mx) for v in lg)
        state, z = splitmix(state)
        u = float(np.float32(z >> 40) * np.float32(1.0 / 16777216.0)) * tot
        acc = 0.0
        for i, v in enumerate(lg):
            acc += math.exp(float(v) - mx)
            if u < acc:
                return i, state
        return len(lg) - 1, state

    rng = np.random.default_rng(7)
    state = 1
    for _ in range(50):
        lg = (rng.standard_normal(512) * 3).astype(np.float32)
        tok, st = alpa.sample_token(lg, True, state)
        assert (tok, st) == ref_sample(lg, state)
        state = st
        assert alpa.sample_token(lg, False, 0)[0] == int(np.argmax(lg))
    bad = np.zeros(8, np.float32)
    bad[3] = np.nan
    with pytest.raises(alpa.InternalError):
        alpa.sample_token(bad, True, 1)
