"""Per-op hardware counters of the persistent iteration kernel from one ncu PM-sampling
capture (tools/ncu_perop.sh): the sampled time series (tensor-pipe %, DRAM %, L2 %)
is cut into the kernel's op windows and averaged per op kind over the 36 blocks.

Op windows: the op plan order (encode, encoder MLP1/MLP2, 36 x [QKV, attention, O, MLP1,
MLP2], head) with each op's share of a block taken from the traced twin's per-op spans
(tools/mk_trace.py output), scaled so the windows tile the captured launch exactly.

    PYTHONPATH=<ncu>/extras/python python tools/pm_ops.py rep.ncu-rep trace.txt [hbm_gbs]
"""
import re
import sys

import numpy as np
import ncu_report

rep, trace = sys.argv[1], sys.argv[2]
hbm_peak = float(sys.argv[3]) if len(sys.argv) > 3 else 6450.9
act = ncu_report.load_report(rep).range_by_idx(0).action_by_idx(0)


def series(name):
    m = act.metric_by_name(name)
    return np.array([m.as_double(i) for i in range(m.num_instances())])


tc = series("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")
dram = series("FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed")
l2 = series("LTS.TriageCompute.lts__throughput.avg.pct_of_peak_sustained_elapsed")
dur_us = act.metric_by_name("gpu__time_duration.sum").as_double() / 1000.0
# the sampled buffer spans more than the launch: keep the samples with active SMs
cyc = series("TPC.TriageCompute.sm__cycles_active.avg")
live = np.nonzero(cyc > 0)[0]
lo, hi = live[0], live[-1] + 1
tc, dram, l2 = tc[lo:hi], dram[lo:hi], l2[lo:hi]
ns = len(tc)
# per-op spans of the traced twin (median column = last field "span")
spans = {}
order = []
for line in open(trace):
    f = line.split()
    if not f or f[0] == "op":
        continue
    try:
        v = float(f[-1])
    except ValueError:
        continue
    order.append(f[0])
    spans.setdefault(f[0], []).append(v)
kinds = ["gemm_qkv", "attention", "gemm_o", "gemm_mlp1", "gemm_mlp2"]
per_block = {k: float(np.median(spans[k])) for k in kinds}
head = [("encode", np.median(spans.get("encode", [3.0]))), ("gemm_enc_mlp1", spans["gemm_enc_mlp1"][0]),
        ("gemm_enc_mlp2", spans["gemm_enc_mlp2"][0])]
plan = head + [(k, per_block[k]) for _ in range(36) for k in kinds] + [("head_update", np.median(spans.get("head_update", [7.0])))]
total = sum(w for _, w in plan)
scale = dur_us / total
t = 0.0
acc = {}
for name, w in plan:
    a, b = int(t * scale / dur_us * ns), int((t + w) * scale / dur_us * ns)
    t += w
    if b <= a:
        continue
    d = acc.setdefault(name, [0, 0.0, 0.0, 0.0, 0.0])
    d[0] += b - a
    d[1] += tc[a:b].sum()
    d[2] += dram[a:b].sum()
    d[3] += l2[a:b].sum()
    d[4] += (b - a) * dur_us / ns
# fold the 36 decoder blocks onto one block period (best-fit period: the sharpest
# folded tensor profile), so the op windows do not drift across blocks
us_per = dur_us / ns
t_blk0 = sum(w for _, w in head) * scale
best = None
for P in np.arange(0.9 * sum(per_block.values()) * scale, 1.1 * sum(per_block.values()) * scale, 0.02):
    for off in np.arange(-3.0, 3.01, 0.25):
        idx = ((t_blk0 + off) + np.arange(36)[:, None] * P + np.arange(int(P))[None, :]) / us_per
        idx = idx.astype(int)
        if idx.max() >= ns:
            continue
        prof = tc[idx].mean(0)
        v = prof.var()
        if best is None or v > best[0]:
            best = (v, P, off, idx)
_, P, off, idx = best
ftc, fdr, fl2 = tc[idx].mean(0), dram[idx].mean(0), l2[idx].mean(0)
# phase: circular shift that best matches a template with the two MLP mainloops
# (the traced twin's dep..mma1 of MLP1 / MLP2) as the busy tensor windows
blk = sum(per_block.values())
L = len(ftc)
tmpl = np.zeros(L)
t0 = 0.0
for k in kinds:
    if k in ("gemm_mlp1", "gemm_mlp2"):
        a, b = int((t0 + 0.5) / blk * P), int((t0 + 0.7 * per_block[k]) / blk * P)
        tmpl[a:b] = 1.0
    t0 += per_block[k]
shift = max(range(L), key=lambda sh: float(np.dot(np.roll(ftc, -sh), tmpl)))
ftc, fdr, fl2 = np.roll(ftc, -shift), np.roll(fdr, -shift), np.roll(fl2, -shift)
fold = {}
t = 0.0
for k in kinds:
    a, b = int(t / blk * P), int((t + per_block[k]) / blk * P)
    t += per_block[k]
    fold[k] = (b - a, ftc[a:b].mean(), fdr[a:b].mean(), fl2[a:b].mean())
print(f"folded block period {P:.2f} us, phase {shift} us (template match on the two MLP mainloops): "
      f"per-op windows at 1 us resolution, block starts at QKV")
print(f"{'op (folded)':16s} {'us/block':>8s} {'tensor%':>8s} {'dram%':>6s} {'dram GB/s':>9s} {'L2%':>5s}")
for k in kinds:
    n, a, b, c = fold[k]
    print(f"{k:16s} {n * us_per:8.1f} {a:8.1f} {b:6.1f} {b / 100 * hbm_peak:9.0f} {c:5.1f}")
print("folded block profile (tensor% per us): " + " ".join(f"{x:.0f}" for x in ftc))
print("folded block profile (dram% per us):   " + " ".join(f"{x:.0f}" for x in fdr))
print()
print(f"launch {dur_us:.1f} us, {ns} PM samples ({dur_us / ns:.2f} us each); windows scaled x{scale:.3f} "
      f"from the traced twin's spans")
print(f"{'op':16s} {'us/launch':>9s} {'us/block':>8s} {'tensor%':>8s} {'dram%':>6s} {'dram GB/s':>9s} {'L2%':>5s}")
for name in ["encode", "gemm_enc_mlp1", "gemm_enc_mlp2"] + kinds + ["head_update"]:
    if name not in acc:
        continue
    n, s_tc, s_dr, s_l2, us = acc[name]
    blocks = 36 if name in kinds else 1
    print(f"{name:16s} {us:9.1f} {us / blocks:8.2f} {s_tc / n:8.1f} {s_dr / n:6.1f} {s_dr / n / 100 * hbm_peak:9.0f} "
          f"{s_l2 / n:5.1f}")
print(f"{'whole launch':16s} {dur_us:9.1f} {'':8s} {tc.mean():8.1f} {dram.mean():6.1f} "
      f"{dram.mean() / 100 * hbm_peak:9.0f} {l2.mean():5.1f}")
