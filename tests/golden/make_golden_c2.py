"""Regenerate tests/golden/expected_c2.npz: config-2-width (Alpamayo-1 action
expert) oracle outputs at the BENCHMARKED depth, so the GPU box can check the
bf16 tensor-core path where it is measured.

Runs ONLY in the dev container.  The checker is the C restatement
(oracle/alpa_oracle.c, ``Port``), which is pinned bitwise to the reference
itself (tests/test_oracle.py: port == oracle/_ref/libminivla_ref.so on the
reference's own configs).  The pin is re-checked here at config-2 width on one
block-iteration against the reference (``Ref``, built from
/root/reference/proj/src) before any fixture is written.

Shape: B=36 blocks, action_hidden_dim 2048 (assumption), kv 1024,
8 heads, r=2048 synthetic prefix (make_sealed_cache recipe seed 4242,
test_model.cpp:43-74), weight_seed 1234, noise seed 2 stride 1.

Cases (keys ``<name>_actions``, ``<name>_traj`` at v0 = 5.0):
  c2_n6_k10     the bench config (BASELINE.json configs[1])
  c2_n1_k10     N=1 (configs[2], the HBM-bound end)
  b2_n64_k2     N=64, B=2, K=2 (configs[2], 3 query tiles of lanes x 8 heads)
  b1_n6_k5 / b1_n6_k20   K sweep at B=1 (configs[3])
  multi_n3_b2_k2  multi topology (lane l -> prefix seed 4242 + 1000 l), B=2, K=2

Usage:  python tests/golden/make_golden_c2.py [--threads 8]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Cfg, Port, Ref, have_ref  # noqa: E402

V0 = 5.0
SEED_PRE = 4242


def c2(B, K):
    return Cfg.make(vision_blocks=0, decoder_blocks=B, hidden_dim=64, action_hidden_dim=2048,
                    kv_dim=1024, heads=8, vocab_size=128, diffusion_iters=K)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--skip-pin", action="store_true")
    args = ap.parse_args()
    port = Port()
    meta = {"v0": V0, "prefix_seed": SEED_PRE, "r": 2048, "cases": {}}

    if not args.skip_pin:
        # port == the reference itself at config-2 width (one block, one iteration)
        if not have_ref():
            raise SystemExit("oracle/_ref/libminivla_ref.so missing: run `make -C oracle`")
        ref = Ref()
        cfg = c2(1, 1)
        pre = port.synthetic_prefix(SEED_PRE, 1, 256, 1024)
        t = time.time()
        a_ref, _, _ = ref.action_generation(cfg, pre, 2)
        a_port = port.refine(cfg, port.weights(cfg), pre, port.noise(2, 1, 2), threads=args.threads)
        assert np.array_equal(a_ref, a_port), "port != reference at config-2 width"
        meta["pin"] = {"case": "B=1 K=1 N=2 r=256 config-2 width", "bitwise_equal": True,
                       "seconds": round(time.time() - t, 1)}
        print("pin: port == reference bitwise at config-2 width", flush=True)

    out = {}
    cases = [
        ("c2_n6_k10", 36, 10, 6, False),
        ("c2_n1_k10", 36, 10, 1, False),
        ("b2_n64_k2", 2, 2, 64, False),
        ("b1_n6_k5", 1, 5, 6, False),
        ("b1_n6_k20", 1, 20, 6, False),
        ("multi_n3_b2_k2", 2, 2, 3, True),
    ]
    weights = {}
    for name, B, K, n, multi in cases:
        cfg = c2(B, K)
        if B not in weights:
            weights.clear()
            weights[B] = port.weights(cfg)
        w = weights[B]
        t = time.time()
        if multi:
            pre = np.stack([port.synthetic_prefix(SEED_PRE + 1000 * l, B, 2048, 1024) for l in range(n)])
            acts = port.refine(cfg, w, pre, port.noise(2, 1, n), lane_prefix=np.arange(n, dtype=np.int32),
                               threads=args.threads)
        else:
            pre = port.synthetic_prefix(SEED_PRE, B, 2048, 1024)
            acts = port.refine(cfg, w, pre, port.noise(2, 1, n), threads=args.threads)
        traj = port.rollout(acts, V0)
        out[f"{name}_actions"] = acts
        out[f"{name}_traj"] = traj
        meta["cases"][name] = {"B": B, "K": K, "n": n, "multi": multi,
                               "actions_fnv": f"{port.fnv1a(acts):016x}",
                               "seconds": round(time.time() - t, 1)}
        print(name, meta["cases"][name], flush=True)
        del pre
    np.savez_compressed(os.path.join(HERE, "expected_c2.npz"), **out)
    with open(os.path.join(HERE, "golden_c2.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
