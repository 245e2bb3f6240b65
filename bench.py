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
    """SM clocks and throttle reasons sampled during the timed region: NVML
    every 5 ms (nvidia-smi every 0.2 s as the fallback)."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.rows = []  # (sm_mhz, max_mhz, reasons set)
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self, nv):
        h = nv.nvmlDeviceGetHandleByIndex(self.device)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        while not self._stop.is_set():
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append((float(sm), float(mx), {k for k, b in bits.items() if r & b}))
            self._stop.wait(0.005)

    def _run_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                f = [x.strip() for x in out.split(",")]
                if len(f) >= 6 and f[0].replace(".", "").isdigit():
                    self.rows.append((float(f[0]), float(f[1]),
                                      {self.NAMES[i] for i in range(4) if f[2 + i].lower() == "active"}))
            except Exception:
                pass
            self._stop.wait(0.2)

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            try:
                self._run_nvml(nv)
            finally:
                nv.nvmlShutdown()
        except Exception:
            self._run_smi()

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
        sm = [r[0] for r in self.rows]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted(set().union(*[r[2] for r in self.rows])), "samples": len(self.rows),
                "sampler": "nvml 5 ms" if len(self.rows) > 3 else "nvidia-smi"}


# ----------------------------------------------------------------------- reference
def _ref_cfg(blocks: int):
    from oracle.oracle import Cfg
    return Cfg.make(vision_blocks=0, hidden_dim=64, vocab_size=128, decoder_blocks=blocks,
                    action_hidden_dim=C2["ah"], kv_dim=C2["kv"], heads=C2["heads"],
                    diffusion_iters=1)


def reference_fit(n: int = C2["n"], variant: str = "best", blocks=(1, 2)):
    """The reference's own CPU path (oracle/_ref, compiled from the reference
    sources; the C restatement, kind "port", if it is missing) on bounded
    samples of the workload: Engine::run_action_generation (noise +
    replicate_for_batch + diffusion_refine, the cli.cpp:273-278 region) at
    full width (ah 2048, kv 1024, r 2048, N lanes), K = 1, for B = 1 and 2
    decoder blocks.  DiffusionResult::iter_ms separates the iteration from the
    per-block replicate, so the scene is assembled term by term:
        per block:  blk = iter(B=2) - iter(B=1)        (one block-iteration)
        encoder+head = iter(B=1) - blk                 (once per iteration)
        replicate per block = rest(B=2) - rest(B=1)    (once per scene)
        scene = rest(B=1) - rep + 36 rep + K (enc + 36 blk)
    variant "best" = static KV + graph executor, "baseline" = dynamic + eager
    (SURVEY §8d)."""
    from oracle.oracle import Port, have_ref, Ref
    port = Port()
    static_kv = graph = variant == "best"
    out = []
    for B in blocks:
        cfg = _ref_cfg(B)
        prefix = port.synthetic_prefix(C2["prefix_seed"], B, C2["r"], C2["kv"])
        if have_ref():
            ref = Ref()
            _, ms, _ = ref.action_generation(cfg, prefix, n, seed=C2["seed"], stride=C2["stride"],
                                             static_kv=static_kv, graph=graph)
            out.append((ms, ref.last_iter_ms))
            kind = "reference"
        else:
            w = port.weights(cfg)
            noise = port.noise(C2["seed"], C2["stride"], n)
            t0 = time.perf_counter()
            port.refine(cfg, w, prefix, noise)
            ms = (time.perf_counter() - t0) * 1e3
            out.append((ms, ms))
            kind = "port"
    res = {"kind": kind, "variant": variant, "n": n, "samples_ms": [o[0] for o in out],
           "sample_iter_ms": [o[1] for o in out]}
    if len(out) == 2:
        (t1, i1), (t2, i2) = out
        blk = max(i2 - i1, 0.0)
        enc = max(i1 - blk, 0.0)
        rep = max((t2 - i2) - (t1 - i1), 0.0)
        base = max((t1 - i1) - rep, 0.0)
        B, K = C2["blocks"], C2["k"]
        res.update(block_iter_ms=blk, enc_head_ms=enc, replicate_per_block_ms=rep, fixed_ms=base,
                   scene_ms=base + B * rep + K * (enc + B * blk))
    else:
        f_s = scene_flops(n, 1, blocks[0], C2["ah"], C2["kv"], C2["r"])
        f_c = scene_flops(C2["n"], C2["k"], C2["blocks"], C2["ah"], C2["kv"], C2["r"])
        res["scene_ms"] = out[0][0] * f_c / f_s
    return res


def cpu_model() -> str:
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def ncores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_sample_subprocess(threads: int, variant: str = "best", n: int = C2["n"], blocks="1,2",
                          timeout: float = 600.0) -> dict:
    """One reference_fit in a child process (OpenMP thread count fixed at its
    start; the GPU arm's process never loads the reference library)."""
    env = dict(os.environ, OMP_NUM_THREADS=str(threads))
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-sample", "--variant",
                          variant, "--sample-n", str(n), "--sample-blocks", blocks],
                         capture_output=True, text=True, env=env, timeout=timeout)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    if out.returncode or not lines:
        raise RuntimeError(f"cpu sample failed: {out.stderr[-400:]}")
    d = json.loads(lines[-1])
    d["threads"] = threads
    return d


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    threads = ncores()
    t_start = time.perf_counter()
    budget_s = 300.0
    fits = []
    if args.warmup > 0:  # page-in, thread pool start
        cpu_sample_subprocess(threads, n=1, blocks="1")
    for _ in range(args.steps):
        t0 = time.perf_counter()
        fits.append(cpu_sample_subprocess(threads))
        if (time.perf_counter() - t_start) + (time.perf_counter() - t0) > budget_s:
            break
    scene_ms = statistics.median(f["scene_ms"] for f in fits)
    traj_s = C2["n"] * 1000.0 / scene_ms
    extra = {}
    try:  # the reference's baseline variant (dynamic KV, eager), one fit
        b = cpu_sample_subprocess(threads, variant="baseline")
        extra["baseline_variant_scene_ms"] = b["scene_ms"]
    except Exception as e:
        extra["baseline_variant_scene_ms"] = f"failed: {e}"
    try:  # one thread, one lane, one block-iteration (bounded), scaled by FLOPs to the scene
        one = cpu_sample_subprocess(1, n=1, blocks="1")
        extra["one_thread_sample_ms"] = one["samples_ms"][0]
        extra["one_thread_scene_ms_flop_scaled"] = one["scene_ms"]
    except Exception as e:
        extra["one_thread_sample_ms"] = f"failed: {e}"
    f0 = fits[0]
    sample_desc = (f"Engine::run_action_generation of the reference ({f0['kind']}, static KV + graph "
                   f"executor) at full width (ah {C2['ah']}, kv {C2['kv']}, r {C2['r']}, N={C2['n']}), "
                   f"K=1, B=1 and B=2; {len(fits)} fits, median scene {scene_ms:.0f} ms assembled from "
                   f"per-block iteration {f0.get('block_iter_ms', 0):.0f} ms, encoder+head "
                   f"{f0.get('enc_head_ms', 0):.0f} ms, replicate {f0.get('replicate_per_block_ms', 0):.0f} "
                   f"ms/block (DiffusionResult::iter_ms) to B=36, K=10")
    line = {
        "impl": "reference", "metric": METRIC, "value": traj_s, "unit": "trajectories/s",
        "n_gpus": world, "steps": len(fits), "warmup": args.warmup,
        "ms_per_step": scene_ms, "ms_per_scene": scene_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_block(args, world),
        "cpu_baseline": {"value": traj_s, "unit": "trajectories/s", "cores": threads,
                         "kind": f0["kind"], "sample": sample_desc, "cpu": cpu_model(), **extra},
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
                     "traffic_src": "profiles/ncu_traffic.json (dram__bytes_read.sum + "
                                    "dram__bytes_write.sum of one iteration launch, ncu --set full)",
                     "algorithmic_bytes_per_launch": per_launch_bytes,
                     "hbm_gbs_algorithmic": per_launch_bytes / (dom_ms * 1e-3) / 1e9,
                     "peak_src": pk["src"],
                     "share_of_step": min(1.0, dom_ms * dom["launches"] / e2e_ms)
                     if dom["name"] == "iteration" and iter_ms else dom["total_ms"] / total_ms,
                     "launches_per_scene": dom["launches"], "ms_per_launch": dom_ms,
                     "timing": dom_src},
        "roofline_path": {"bound": "tensor" if F / (pk["tc"] * 1e12) > Bm / (pk["hbm"] * 1e9)
                          else "hbm", "t_roof_ms": t_roof, "t_measured_ms": ms,
                          "frac": t_roof / ms, "tflop_per_scene": F / 1e12,
                          "min_gb_per_scene": Bm / 1e9, "peak_src": pk["src"]},
        # NOT the timed run: one eager scene of the instrumented twin (a sync per
        # launch, globaltimer stamps), for the per-op breakdown only
        "diagnostics": {
            "source": "alpa_profile: one eager scene of the instrumented twin kernel (sync per "
                      "launch), not the timed graphs",
            "kernels": {p["name"]: {"ms_per_scene": p["total_ms"], "launches": p["launches"],
                                    "tflops": p["flops"] / max(p["total_ms"], 1e-9) / 1e9,
                                    "gbs_algorithmic": p["bytes"] / max(p["total_ms"], 1e-9) / 1e6}
                        for p in prof},
            "op_spans": {p["name"][5:]: {"ms_per_scene": p["total_ms"], "count": p["launches"],
                                          "tflops": p["flops"] / max(p["total_ms"], 1e-9) / 1e9}
                         for p in spans}},
        "gpu_launches": gpu_launches,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_sweeps:
        line["sweeps"] = run_sweeps(gen, stream, pk)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_sample_subprocess(ncores())
            line["cpu_baseline"] = {
                "value": C2["n"] * 1000.0 / cb["scene_ms"], "unit": "trajectories/s",
                "cores": ncores(), "kind": cb["kind"], "cpu": cpu_model(),
                "sample": (f"reference Engine::run_action_generation (static KV, graph executor) "
                           f"at full width, N={C2['n']}, K=1, B=1 and B=2 "
                           f"({cb['samples_ms'][0]:.0f} + {cb['samples_ms'][1]:.0f} ms, child "
                           f"process); scene {cb['scene_ms']:.0f} ms assembled per term (block "
                           f"iteration x36 x10, encoder+head x10, replicate x36) from "
                           f"DiffusionResult::iter_ms")}
        except Exception as e:  # reported, never fatal for the GPU number
            line["cpu_baseline"] = {"value": None, "unit": "trajectories/s", "cores": ncores(),
                                    "kind": "reference", "sample": f"failed: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    gen.close()


SWEEPS = [("N", 1, 10), ("N", 16, 10), ("N", 64, 10), ("K", 6, 5), ("K", 6, 20), ("K", 6, 50)]


def run_sweeps(gen, stream, pk, warm: int = 2, reps: int = 3):
    """BASELINE configs[2] (N = 1/16/64) and configs[3] (K = 5/20/50) on the
    same context and prefix: the whole K loop + rollout as one graph per scene,
    inputs resident, CUDA events on the library's stream.  Each row: ms/scene,
    trajectories/s and its roofline (T_roof / T_measured with the SURVEY §8d
    work and byte counts of that config; at N = 1 the bound is HBM, reported as
    achieved GB/s of the minimum bytes)."""
    import torch
    import paper_2605_08975_b200 as alpa
    rows = []
    for kind, n, K in SWEEPS:
        req = alpa.InferenceRequest(num_trajectories=n, diffusion_iters=K, action_init_seed=C2["seed"],
                                    action_seed_stride=C2["stride"], v0=C2["v0"])
        noise = torch.from_numpy(alpa.host_noise(C2["seed"], C2["stride"], n)).cuda()
        acts = torch.empty((n, 64, 2), dtype=torch.float32, device="cuda")
        traj = torch.empty((n, 64, 3), dtype=torch.float32, device="cuda")
        for _ in range(warm):
            gen.generate_device(req, noise.data_ptr(), acts.data_ptr(), traj.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            gen.generate_device(req, noise.data_ptr(), acts.data_ptr(), traj.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        F = scene_flops(n, K, C2["blocks"], C2["ah"], C2["kv"], C2["r"])
        Bm = scene_bytes(n, K, C2["blocks"], C2["ah"], C2["kv"], C2["r"])
        t_tc, t_hbm = F / (pk["tc"] * 1e12) * 1e3, Bm / (pk["hbm"] * 1e9) * 1e3
        row = {"sweep": kind, "n": n, "k": K, "ms_per_scene": ms, "trajectories_per_s": n * 1000.0 / ms,
               "tflops": F / (ms * 1e-3) / 1e12, "bound": "tensor" if t_tc >= t_hbm else "hbm",
               "t_roof_ms": max(t_tc, t_hbm), "frac": max(t_tc, t_hbm) / ms,
               "finite": bool(torch.isfinite(acts).all().item())}
        if row["bound"] == "hbm":
            row["hbm_gbs"] = Bm / (ms * 1e-3) / 1e9
            row["hbm_frac"] = row["hbm_gbs"] / pk["hbm"]
        rows.append(row)
    return rows


def run_batched(args, rank, world, local_rank):
    """BASELINE configs[4]: `--scenes S` scenes x N=`--n` trajectories, scenes
    round-robin over the ranks (paper_2605_08975_b200.dist.run_scenes): the
    root produces each scene's prefix (the synthetic stand-in for the
    reasoning stage) and sends it to the owner over NCCL P2P on a side stream
    (overlapping the owner's denoise of its previous scene); trajectories are
    all-gathered once.  A step = the whole batch; strong scaling."""
    import torch
    import torch.distributed as dist
    import paper_2605_08975_b200 as alpa
    from paper_2605_08975_b200 import dist as pdist

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if world == 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    n, K, S = args.n, C2["k"], args.scenes
    cfg = alpa.ModelConfig(vision_blocks=0, hidden_dim=64, vocab_size=128,
                           decoder_blocks=C2["blocks"], action_hidden_dim=C2["ah"],
                           kv_dim=C2["kv"], heads=C2["heads"], diffusion_iters=K,
                           weight_seed=C2["weight_seed"], dtype="bf16")
    gen = alpa.ActionGenerator(cfg, device=local_rank)
    stream = torch.cuda.Stream(dev)
    side = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    gen.set_stream(stream.cuda_stream)
    per = gen.prefix_bytes(C2["r"])
    req = alpa.InferenceRequest(num_trajectories=n, action_init_seed=C2["seed"],
                                action_seed_stride=C2["stride"], v0=C2["v0"])
    noise = torch.from_numpy(alpa.host_noise(C2["seed"], C2["stride"], n)).to(dev)

    def make_buf():
        return torch.empty(per // 2, dtype=torch.bfloat16, device=dev)

    def produce(s, buf):
        gen.synthesize_prefix(buf.data_ptr(), C2["prefix_seed"] + 1000 * s, C2["r"])

    def compute(s, buf):
        gen.bind_prefix_device(buf.data_ptr(), 1, C2["r"])
        acts = torch.empty((n, 64, 2), dtype=torch.float32, device=dev)
        traj = torch.empty((n, 64, 3), dtype=torch.float32, device=dev)
        gen.generate_device(req, noise.data_ptr(), acts.data_ptr(), traj.data_ptr())
        return traj

    def batch():
        return pdist.run_scenes(S, compute, produce, make_buf, side_stream=side)

    for _ in range(args.warmup):
        batch()
    torch.cuda.synchronize(dev)
    dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            full, mine = batch()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    pk = peaks()
    F = S * scene_flops(n, K, C2["blocks"], C2["ah"], C2["kv"], C2["r"])
    line = {
        "metric": METRIC, "value": S * n * 1000.0 / ms, "unit": "trajectories/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "ms_per_scene": ms / S,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (scene s prefix seed 4242 + 1000 s, splitmix64 weights seed 1234)",
        "config": {"workload": f"batched scenes (configs[4]): {S} scenes x N={n} trajectories x K={K}, "
                               f"scenes round-robin over {world} GPU(s), prefix P2P from the producing "
                               f"rank + one trajectory all-gather",
                   "scenes": S, "trajectories_per_scene": n, "blocks": C2["blocks"],
                   "action_hidden_dim": C2["ah"], "kv_dim": C2["kv"], "prefix_tokens": C2["r"],
                   "parallelism": f"scene-sharded x{world}",
                   "l2": "inputs larger than L2 (3.1 GB weights + 302 MB prefix per scene)"},
        "roofline_path": {"t_roof_ms": F / (pk["tc"] * 1e12) * 1e3 / world, "t_measured_ms": ms,
                          "frac": F / (pk["tc"] * 1e12) * 1e3 / world / ms, "bound": "tensor",
                          "peak_src": pk["src"]},
        "finite": bool(torch.isfinite(full).all().item()),
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    gen.close()


def _free_port() -> int:
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweeps", action="store_true")
    ap.add_argument("--scenes", type=int, default=0, help="configs[4] batched-scene mode")
    ap.add_argument("--n", type=int, default=16, help="trajectories per scene (--scenes mode)")
    # internal: one bounded reference sample in a child process (cpu_baseline legs)
    ap.add_argument("--cpu-sample", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--variant", default="best", help=argparse.SUPPRESS)
    ap.add_argument("--sample-n", type=int, default=C2["n"], help=argparse.SUPPRESS)
    ap.add_argument("--sample-blocks", default="1,2", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.cpu_sample:
        blocks = tuple(int(b) for b in args.sample_blocks.split(","))
        print(json.dumps(reference_fit(args.sample_n, args.variant, blocks)), flush=True)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` launches its own N ranks (one per GPU)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.run(cmd).returncode)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"note: WORLD_SIZE={world} overrides --gpus {args.gpus}", file=sys.stderr)
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.scenes:
            run_batched(args, rank, world, local_rank)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
