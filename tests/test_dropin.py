"""The reference engine itself with its action stage routed to the B200 library
(include/alpa_minivla_adapter.hpp): tests/cpp/ref_dropin.cpp linked against the
reference's own objects (compiled from /root/reference/proj/src by
oracle/Makefile; the prebuilt binary travels to the GPU box as
oracle/_ref/ref_dropin).

GPU: for single/multi topology x N in {1, 6} x the three compare-actiongen
variants (cli.cpp:236-313) the drop-in reproduces Engine::infer's actions and
trajectories (rel-L2 <= 1e-4, fp32 path), the device rollout equals the
reference's host rollout bitwise, the variants are bitwise equal, kv_bytes
matches LatencyReport::kv_bytes, and the reference's exception types come back
for N = 0, a mismatched multi cache and graph + dynamic.
"""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "ref_dropin")
HDR = os.path.join(ROOT, "include", "alpa_minivla_adapter.hpp")


def test_adapter_builds_against_reference_headers():
    """Builds wherever the reference sources exist (the dev container); on the
    GPU box the prebuilt binary must have travelled."""
    if not os.path.isdir("/root/reference/proj/include"):
        assert os.path.exists(EXE), "oracle/_ref/ref_dropin missing (build it with make -C oracle)"
        return
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "_ref/ref_dropin"], check=True)
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_reference_engine_with_gpu_action_stage():
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    for l in lines:
        print(l)
    assert out.returncode == 0, out.stderr + out.stdout
    cases = [l for l in lines if "variant" in l]
    errors = [l for l in lines if "error_case" in l]
    reasoning = [l for l in lines if l.get("device_reasoning")]
    assert len(cases) == 12 and all(c["pass"] for c in cases)
    assert len(errors) == 3 and all(e["pass"] for e in errors)
    assert len(reasoning) == 4 and all(c["pass"] for c in reasoning)
