"""The C++ drop-in: a reference-style caller compiled against
include/alpa_minivla_shim.hpp and linked to libalpa_action.so.

CPU: it compiles and links (no compute).  GPU: it reproduces the golden
config-1 actions / trajectories and maps errors to the reference exit codes.
"""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2605_08975_b200")


def build_demo(tmp_path):
    exe = str(tmp_path / "shim_demo")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_demo.cpp"), "-L", PKG,
                    "-lalpa_action", f"-Wl,-rpath,{PKG}", "-o", exe], check=True)
    return exe


def test_shim_compiles_and_links(tmp_path):
    exe = build_demo(tmp_path)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_shim_reproduces_golden(tmp_path, golden):
    exe = build_demo(tmp_path)
    pre = tmp_path / "prefix.bin"
    golden["prefix"].astype(np.float32).tofile(pre)
    oa, ot = tmp_path / "a.bin", tmp_path / "t.bin"
    r = golden["prefix"].shape[2]
    out = subprocess.run([exe, str(pre), str(r), "6", str(oa), str(ot)], capture_output=True,
                         text=True)
    assert out.returncode == 0, out.stderr
    acts = np.fromfile(oa, np.float32).reshape(6, 64, 2)
    traj = np.fromfile(ot, np.float32).reshape(6, 64, 3)
    ea, et = golden["expected"]["n6_k10_actions"], golden["expected"]["n6_k10_traj"]
    assert np.linalg.norm(acts - ea) / np.linalg.norm(ea) <= 1e-4
    assert np.linalg.norm(traj - et) / np.linalg.norm(et) <= 1e-4
    lines = {ln.split(" ", 1)[0]: ln.split(" ", 1)[1] for ln in out.stdout.splitlines() if " " in ln}
    # open-loop metrics through the shim == the C restatement of eval.cpp, bitwise
    from oracle.oracle import Port, Ref, have_ref
    port = Port()
    m = dict(kv.split("=") for kv in lines["metrics"].split())
    assert float(m["min_ade"]) == port.min_ade(traj, traj[0])
    assert float(m["diversity"]) == port.diversity(traj)
    # LatencyReport wire format: parsed by the reference's own from_json
    rep = json.loads(lines["report"])
    assert len(rep["action_gen_iter_ms"]) == 10 and rep["action_gen_ms"] > 0
    assert rep["replay_count"] == 1 and rep["alloc_count"] == 0
    if have_ref():
        n_iter, ms = Ref().parse_latency_report(lines["report"])
        assert n_iter == 10 and ms == rep["action_gen_ms"]
    # N = 0 -> ConfigError -> exit code 2 (pipeline.cpp:203-205, cli.cpp:528-540)
    bad = subprocess.run([exe, str(pre), str(r), "0", str(oa), str(ot)], capture_output=True)
    assert bad.returncode == 2
    # missing prefix file -> IoError -> exit code 1
    bad = subprocess.run([exe, str(tmp_path / "nope.bin"), str(r), "6", str(oa), str(ot)],
                         capture_output=True)
    assert bad.returncode == 1


@pytest.mark.gpu
def test_shim_device_reasoning_stage(tmp_path, golden):
    """Engine::run_reasoning_device (the LM prefill/decode + KV on the device,
    reference sampler) then the action stage on the in-place KV: the demo
    scenario's actions / trajectories match the reference's (golden config 1),
    and the LatencyReport carries the reasoning components and CoT length."""
    exe = build_demo(tmp_path)
    rz = np.load(os.path.join(ROOT, "tests", "golden", "reasoning_c1.npz"))
    vis, prompt = tmp_path / "vision.bin", tmp_path / "prompt.bin"
    rz["vision"].astype(np.float32).tofile(vis)
    rz["prompt"].astype(np.int64).tofile(prompt)
    oa, ot = tmp_path / "a.bin", tmp_path / "t.bin"
    out = subprocess.run([exe, "--reason", str(vis), str(rz["vision"].shape[0]), str(prompt), "6", str(oa),
                          str(ot)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    acts = np.fromfile(oa, np.float32).reshape(6, 64, 2)
    traj = np.fromfile(ot, np.float32).reshape(6, 64, 3)
    ea, et = golden["expected"]["n6_k10_actions"], golden["expected"]["n6_k10_traj"]
    assert np.linalg.norm(acts - ea) / np.linalg.norm(ea) <= 1e-4
    assert np.linalg.norm(traj - et) / np.linalg.norm(et) <= 1e-4
    lines = {ln.split(" ", 1)[0]: ln.split(" ", 1)[1] for ln in out.stdout.splitlines() if " " in ln}
    assert lines["reasoning"] == f"r={int(rz['r'])} steps={int(rz['m'])}"
    rep = json.loads(lines["report"])
    assert rep["reasoning_prefill_ms"] > 0 and rep["reasoning_decode_ms"] > 0
    assert rep["cot_tokens"] == int(rz["m"]) - 1 and rep["action_gen_ms"] > 0
