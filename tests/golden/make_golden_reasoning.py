"""Regenerate tests/golden/reasoning_c1.npz from the reference itself (dev
container only: needs oracle/_ref/libminivla_ref.so built from /root/reference).

The reasoning stage of config 1 (fixtures/default_config.json model, demo
scenario, single topology, stochastic sampler seed 1), as the device KV
producer (paper_2605_08975_b200 reasoning_*) consumes and
produces it:

* vision      [P][hidden] f32  Model::vision_encode of the request's patch rows
                               (model.cpp:326-392, pipeline.cpp:265-277)
* prompt      [n] int64        Engine::preprocess prompt token ids
* decode_ids  [m] int64        the ids the decode loop fed back (cot tokens +
                               the terminator, pipeline.cpp:345-386)
* prefix      [B][2][r][kv]    the sealed reasoning KV (Engine::run_reasoning)
* T, m, r, fingerprint, v0     scalars (KvCache::reasoning_fingerprint, kv_cache.cpp:346)

Usage:  python tests/golden/make_golden_reasoning.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Cfg, Ref  # noqa: E402

SCENARIO = "/root/reference/proj/fixtures/demo_scenario.json"


def main():
    ref = Ref()
    cfg = Cfg.make()
    vis, prompt, ids, T, m = ref.reasoning_io(cfg, SCENARIO, sampler_seed=1, stochastic=True)
    prefix, fp, v0 = ref.scenario_prefix(cfg, SCENARIO)
    assert prefix.shape[2] == T + m, (prefix.shape, T, m)
    np.savez_compressed(os.path.join(HERE, "reasoning_c1.npz"), vision=vis, prompt=prompt, decode_ids=ids,
                        prefix=prefix, T=T, m=m, r=prefix.shape[2], fingerprint=np.uint64(fp), v0=v0)
    print(f"P={vis.shape[0]} prompt={prompt.size} T={T} m={m} r={prefix.shape[2]} fingerprint={fp:016x}")


if __name__ == "__main__":
    main()
