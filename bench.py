#!/usr/bin/env python
"""Benchmark of the single-reasoning diffusion action-generation hot path.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): one scene =
one shared synthetic 2048-token reasoning prefix (make_sealed_cache recipe,
seed 4242) conditioning N=6 trajectories through K=10 denoising iterations of
an Alpamayo-1-width action expert (36 blocks, action_hidden_dim 2048 [SURVEY
assumption], kv 1024, 8 heads), bf16 tensor cores, followed by the rollout.
Weights are random-init from the reference's splitmix64 stream (seed 1234).

A "step" is one scene.  `value` = trajectories/s over all ranks with inputs
resident in HBM (alpa_generate_device), `e2e` = the same through the public
host-buffer call (alpa_generate: host noise + H2D + refine + rollout + D2H).
Multi-GPU (torchrun): each step the root produces the scene prefix, NCCL
broadcasts it (302 MB), every rank denoises its own N=6 lanes of the scene
(global lane indices keep the noise seeds) and the actions are all-gathered:
weak scaling in trajectories.

The inputs are larger than L2 (3.1 GB of weights + 302 MB prefix streamed per
scene), so no explicit L2 flush is needed between timed steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("diffusion action-gen latency ms/scene (N traj × K steps); "
          "trajectories/sec @1/2/4/8")

C2 = dict(blocks=36, ah=2048, kv=1024, heads=8, r=2048, n=6, k=10, prefix_seed=4242,
          weight_seed=1234, seed=2, stride=1, v0=5.0)


def scene_flops(n, k, B, ah, kv, r, A=64):
    """algorithmic FLOPs of one scene."""
    M = 64 * n
    per_iter = (2 * M * 2 * ah + 16 * M * ah * ah +
                B * (6 * M * ah * kv + 4 * n * A * (r + A) * kv + 2 * M * kv * ah +
                     16 * M * ah * ah) + 4 * M * ah)
    return k * per_iter


def scene_bytes(n, k, B, ah, kv, r, A=64, eb=2):
    """minimum HBM bytes of one scene (weights once per
    iteration, shared prefix once, action K/V write+read)."""
    per_iter = (eb * (8 * ah * ah + 2 * ah + B * (4 * ah * kv + 8 * ah * ah) + 2 * ah) +
                B * 2 * r * kv * eb + B * 2 * n * A * kv * eb * 2)
    return k * per_iter


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm": p["hbm_gbs"], "tc": p["bf16_tflops"], "tc_sustained":
                p.get("bf16_tflops_sustained", p["bf16_tflops"]), "src": "measured"}
    except Exception:
        return {"hbm": 6650.0, "tc": 1590.0, "tc_sustained": 1400.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ----------------------------------------------------------------------- reference
def reference_sample(threads: int | None = None, n: int = C2["n"]):
    """Time the reference's own CPU path (oracle/_ref, compiled from the
    reference sources) on a bounded sample of the workload: Engine::
    run_action_generation (replicate + host noise + diffusion_refine,
    cli.cpp:273-278 region) for ONE decoder block and ONE iteration at full
    width (ah 2048, kv 1024, r 2048, N lanes).  Scene time is extrapolated by
    the algorithmic FLOP ratio (the reference runs at a constant GFLOP/s).
    Falls back to the C restatement (kind "port") if the reference library
    is missing."""
    import numpy as np
    from oracle.oracle import Cfg, Port, have_ref, Ref
    if threads:
        os.environ["OMP_NUM_THREADS"] = str(threads)
    port = Port()
    cfg = Cfg.make(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=1,
                   action_hidden_dim=C2["ah"], kv_dim=C2["kv"], heads=C2["heads"],
                   diffusion_iters=1)
    prefix = port.synthetic_prefix(C2["prefix_seed"], 1, C2["r"], C2["kv"])
    f_sample = scene_flops(n, 1, 1, C2["ah"], C2["kv"], C2["r"])
    f_scene = scene_flops(C2["n"], C2["k"], C2["blocks"], C2["ah"], C2["kv"], C2["r"])
    if have_ref():
        ref = Ref()
        t0 = time.perf_counter()
        _, ms, _ = ref.action_generation(cfg, prefix, n, seed=C2["seed"], stride=C2["stride"])
        wall = (time.perf_counter() - t0) * 1e3
        kind = "reference"
    else:
        w = port.weights(cfg)
        noise = port.noise(C2["seed"], C2["stride"], n)
        t0 = time.perf_counter()
        port.refine(cfg, w, prefix, noise)
        ms = (time.perf_counter() - t0) * 1e3
        wall = ms
        kind = "port"
    return {"sample_ms": ms, "scene_ms": ms * f_scene / f_sample, "kind": kind,
            "wall_ms": wall, "f_ratio": f_scene / f_sample}


def ncores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    threads = ncores()
    samples = []
    # warm-up: a cheap N=1 sample per requested warm-up step (page-in, threads)
    for _ in range(max(args.warmup, 1) if args.warmup < 3 else 1):
        reference_sample(threads, n=1)
    budget_s, est = 240.0, None
    for i in range(args.steps):
        t0 = time.perf_counter()
        samples.append(reference_sample(threads))
        est = time.perf_counter() - t0
        if (i + 1) * est > budget_s:
            break
    scene_ms = statistics.median(s["scene_ms"] for s in samples)
    traj_s = C2["n"] * 1000.0 / scene_ms
    kind = samples[0]["kind"]
    sample_desc = (f"Engine::run_action_generation of the reference ({kind}) on 1 decoder block x "
                   f"1 iteration at full width (ah {C2['ah']}, kv {C2['kv']}, r {C2['r']}, "
                   f"N={C2['n']}), {len(samples)} timed samples, median "
                   f"{statistics.median(s['sample_ms'] for s in samples):.0f} ms; scene time "
                   f"extrapolated x{samples[0]['f_ratio']:.1f} by algorithmic FLOPs to B=36, K=10")
    line = {
        "impl": "reference", "metric": METRIC, "value": traj_s, "unit": "trajectories/s",
        "n_gpus": world, "steps": len(samples), "warmup": args.warmup,
        "ms_per_step": scene_ms, "ms_per_scene": scene_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_block(args, world),
        "cpu_baseline": {"value": traj_s, "unit": "trajectories/s", "cores": threads,
                         "kind": kind, "sample": sample_desc},
        "e2e": {"value": traj_s, "unit": "trajectories/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_block(args, world):
    return {"workload": (f"alpamayo1-width action expert, single-reasoning scene: one shared "
                         f"{C2['r']}-token prefix KV, N={C2['n']} trajectories/GPU x K={C2['k']} "
                         f"denoising steps + rollout"),
            "blocks": C2["blocks"], "action_hidden_dim": C2["ah"], "kv_dim": C2["kv"],
            "heads": C2["heads"], "prefix_tokens": C2["r"], "trajectories_per_gpu": C2["n"],
            "trajectories_total": C2["n"] * world, "diffusion_steps": C2["k"],
            "parallelism": f"dp{world} (trajectory slices of one scene, NCCL prefix broadcast "
                           f"+ action all-gather)" if world > 1 else "single GPU",
            "l2": "inputs larger than L2 (3.1 GB weights + 302 MB prefix per scene)"}


# ----------------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import paper_2605_08975_b200 as alpa

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
    n, K = C2["n"], C2["k"]
    cfg = alpa.ModelConfig(vision_blocks=0, hidden_dim=64, vocab_size=128,
                           decoder_blocks=C2["blocks"], action_hidden_dim=C2["ah"],
                           kv_dim=C2["kv"], heads=C2["heads"], diffusion_iters=K,
                           weight_seed=C2["weight_seed"], dtype="bf16")
    gen = alpa.ActionGenerator(cfg, device=local_rank)
    # a dedicated (non-default) stream shared by torch events, NCCL and the library
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    gen.set_stream(stream.cuda_stream)
    pre_bytes = gen.prefix_bytes(C2["r"])
    prefix = torch.empty(pre_bytes // 2, dtype=torch.bfloat16, device=dev)
    if rank == 0:
        gen.synthesize_prefix(prefix.data_ptr(), C2["prefix_seed"], C2["r"])
    if dist is not None:
        dist.broadcast(prefix, 0)
    gen.bind_prefix_device(prefix.data_ptr(), 1, C2["r"])
    lane0 = rank * n
    req = alpa.InferenceRequest(num_trajectories=n, lane0=lane0, action_init_seed=C2["seed"],
                                action_seed_stride=C2["stride"], v0=C2["v0"])
    noise = torch.from_numpy(alpa.host_noise(C2["seed"], C2["stride"], n, lane0)).to(dev)
    acts = torch.empty((n, 64, 2), dtype=torch.float32, device=dev)
    traj = torch.empty((n, 64, 3), dtype=torch.float32, device=dev)
    from paper_2605_08975_b200 import dist as pdist

    def step(scene: int):
        if dist is not None:
            # the scene's prefix: produced on the root, one NCCL broadcast
            if rank == 0:
                gen.synthesize_prefix(prefix.data_ptr(), C2["prefix_seed"] + 1000 * scene,
                                      C2["r"])
            pdist.broadcast_prefix(prefix, 0)
        gen.generate_device(req, noise.data_ptr(), acts.data_ptr(), traj.data_ptr())
        if dist is not None:
            pdist.gather_lanes(acts, world * n)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for i in range(args.steps):
            step(i)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * n * 1000.0 / ms

    # end to end through the public host-buffer API
    if dist is not None:
        gen.bind_prefix_device(prefix.data_ptr(), 1, C2["r"])
    for _ in range(max(1, args.warmup)):
        gen.run_action_generation(req)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    st = None
    iter_ms = []  # per-iteration device times (CUDA event nodes inside the scene's graph)
    for _ in range(args.steps):
        res = gen.run_action_generation(req)
        st = res.stats
        iter_ms += list(st.get("iter_ms") or [])
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    if dist is not None:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": world * n * 1000.0 / e2e_ms, "unit": "trajectories/s",
           "ms_per_scene": e2e_ms, "h2d_bytes_per_step": int(st["h2d_bytes"]) + 4 + 4 * n,
           "d2h_bytes_per_step": int(st["d2h_bytes"]) + 4}

    # per-kernel breakdown (CUDA events around each launch of one eager scene)
    allprof = gen.profile(req, iters=K)
    # "span:<op>" entries are per-op spans inside the persistent iteration
    # kernel (globaltimer stamps), not separate launches
    prof = [p for p in allprof if not p["name"].startswith("span:")]
    spans = [p for p in allprof if p["name"].startswith("span:")]
    pk = peaks()
    total_ms = sum(p["total_ms"] for p in prof)
    dom = max(prof, key=lambda p: p["total_ms"])
    tensor_kernels = ("gemm", "attention", "iteration")
    bound = "tensor" if dom["name"].startswith(tensor_kernels) else "hbm"
    # the dominant kernel's average launch duration: for the persistent iteration
    # kernel, CUDA events recorded between the iterations inside the production
    # graph during the timed e2e scenes; otherwise the eager per-launch profile
    dom_ms = dom["total_ms"] / max(dom["launches"], 1)
    dom_src = "eager per-launch CUDA events (alpa_profile)"
    if dom["name"] == "iteration" and iter_ms:
        dom_ms = sum(iter_ms) / len(iter_ms)
        dom_src = f"CUDA event nodes between iterations in the timed graphs ({len(iter_ms)} launches)"
    per_launch_flops = dom["flops"] / max(dom["launches"], 1)
    per_launch_bytes = dom["bytes"] / max(dom["launches"], 1)
    if bound == "tensor":
        ach = per_launch_flops / (dom_ms * 1e-3) / 1e12
        peak, unit = pk["tc"], "TFLOP/s"
    else:
        ach = per_launch_bytes / (dom_ms * 1e-3) / 1e9
        peak, unit = pk["hbm"], "GB/s"
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(dom["name"])
    except Exception:
        pass
    F = scene_flops(n, K, C2["blocks"], C2["ah"], C2["kv"], C2["r"])
    Bm = scene_bytes(n, K, C2["blocks"], C2["ah"], C2["kv"], C2["r"])
    t_roof = max(F / (pk["tc"] * 1e12), Bm / (pk["hbm"] * 1e9)) * 1e3
    gpu_launches = int(st["graph_nodes"]) * args.steps if st else None

    line = {
        "metric": METRIC, "value": value, "unit": "trajectories/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "ms_per_scene": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (make_sealed_cache prefix seed 4242, splitmix64 weights seed 1234)",
        "config": config_block(args, world),
        "e2e": e2e,
        "roofline": {"bound": bound, "kernel": dom["name"], "achieved": ach, "peak": peak,
                     "unit": unit, "frac": ach / peak, "traffic": traffic,
                     "peak_src": pk["src"],
                     "share_of_step": min(1.0, dom_ms * dom["launches"] / e2e_ms)
                     if dom["name"] == "iteration" and iter_ms else dom["total_ms"] / total_ms,
                     "launches_per_scene": dom["launches"], "ms_per_launch": dom_ms,
                     "timing": dom_src},
        "roofline_path": {"bound": "tensor" if F / (pk["tc"] * 1e12) > Bm / (pk["hbm"] * 1e9)
                          else "hbm", "t_roof_ms": t_roof, "t_measured_ms": ms,
                          "frac": t_roof / ms, "tflop_per_scene": F / 1e12,
                          "min_gb_per_scene": Bm / 1e9, "peak_src": pk["src"]},
        "kernels": {p["name"]: {"ms_per_scene": p["total_ms"], "launches": p["launches"],
                                "tflops": p["flops"] / max(p["total_ms"], 1e-9) / 1e9,
                                "gbs": p["bytes"] / max(p["total_ms"], 1e-9) / 1e6}
                    for p in prof},
        "op_spans": {p["name"][5:]: {"ms_per_scene": p["total_ms"], "count": p["launches"],
                                      "tflops": p["flops"] / max(p["total_ms"], 1e-9) / 1e9}
                     for p in spans},
        "gpu_launches": gpu_launches,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = reference_sample(ncores())
            line["cpu_baseline"] = {
                "value": C2["n"] * 1000.0 / cb["scene_ms"], "unit": "trajectories/s",
                "cores": ncores(), "kind": cb["kind"],
                "sample": (f"reference Engine::run_action_generation, 1 block x 1 iteration at "
                           f"full width, N={C2['n']}: {cb['sample_ms']:.0f} ms, extrapolated "
                           f"x{cb['f_ratio']:.1f} by FLOPs to one scene ({cb['scene_ms']:.0f} ms)")}
        except Exception as e:  # reported, never fatal for the GPU number
            line["cpu_baseline"] = {"value": None, "unit": "trajectories/s", "cores": ncores(),
                                    "kind": "reference", "sample": f"failed: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    gen.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
