"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracle.

Two checkers live behind this module:

* ``Port``  — ``oracle/_ref/liboracle_port.so``, the plain-C restatement
  (``oracle/alpa_oracle.c``) of the reference path.  Always buildable
  (``make -C oracle``), travels to the GPU box as a prebuilt ``.so``.
* ``Ref``   — ``oracle/_ref/libminivla_ref.so``, the reference itself compiled
  from ``/root/reference/proj/src`` by ``oracle/Makefile`` plus the thin
  ``oracle/ref_driver.cpp`` call shim.  Built in the dev container; the
  prebuilt ``.so`` travels to the GPU box.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  The product package
(``paper_2605_08975_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
PORT_SO = os.path.join(REF_DIR, "liboracle_port.so")
REF_SO = os.path.join(REF_DIR, "libminivla_ref.so")

_f32p = C.POINTER(C.c_float)
_i32p = C.POINTER(C.c_int32)


def build() -> None:
    """Compile the C restatement (and the reference when its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


def _fp(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(_f32p)


class Cfg(C.Structure):
    """ModelConfig (include/minivla/model.hpp:12-29); same field order as
    ``orc_cfg`` (alpa_oracle.h) and ``RefCfg`` (ref_driver.cpp)."""

    _fields_ = [
        ("vision_blocks", C.c_int64),
        ("decoder_blocks", C.c_int64),
        ("hidden_dim", C.c_int64),
        ("action_hidden_dim", C.c_int64),
        ("kv_dim", C.c_int64),
        ("heads", C.c_int64),
        ("vocab_size", C.c_int64),
        ("patch_size", C.c_int64),
        ("action_steps", C.c_int64),
        ("diffusion_iters", C.c_int64),
        ("max_new_tokens", C.c_int64),
        ("update_scale", C.c_float),
        ("weight_seed", C.c_uint64),
    ]

    @classmethod
    def make(cls, **kw) -> "Cfg":
        d = dict(vision_blocks=4, decoder_blocks=6, hidden_dim=64, action_hidden_dim=32,
                 kv_dim=32, heads=4, vocab_size=512, patch_size=14, action_steps=64,
                 diffusion_iters=10, max_new_tokens=256, update_scale=0.1, weight_seed=1234)
        d.update(kw)
        return cls(**d)

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class _Linear(C.Structure):
    _fields_ = [("w", _f32p), ("b", _f32p), ("in_", C.c_int64), ("out", C.c_int64)]


class _Weights(C.Structure):
    _fields_ = [("arena", _f32p), ("count", C.c_int64), ("action_in", _Linear),
                ("mlp1", _Linear), ("mlp2", _Linear), ("head", _Linear),
                ("blocks", C.POINTER(_Linear))]


class Port:
    """The C restatement (alpa_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_action_stream_offset.restype = C.c_int64
        L.orc_action_stream_offset.argtypes = [C.POINTER(Cfg)]
        L.orc_action_param_count.restype = C.c_int64
        L.orc_action_param_count.argtypes = [C.POINTER(Cfg)]
        L.orc_weights_build.argtypes = [C.POINTER(Cfg), C.POINTER(_Weights)]
        L.orc_weights_free.argtypes = [C.POINTER(_Weights)]
        L.orc_noise.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, C.c_int64, _f32p]
        L.orc_synthetic_prefix.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, _f32p]
        L.orc_sinusoidal_table.argtypes = [C.c_int64, C.c_int64, _f32p]
        L.orc_diffusion_refine.argtypes = [C.POINTER(Cfg), C.POINTER(_Weights), _f32p, C.c_int64,
                                           _i32p, C.c_int64, C.c_int64, _f32p, C.c_int]
        L.orc_rollout.argtypes = [_f32p, C.c_int64, C.c_int64, C.c_float, _f32p]
        L.orc_min_ade.argtypes = [_f32p, C.c_int64, C.c_int64, _f32p, C.POINTER(C.c_double)]
        L.orc_diversity.argtypes = [_f32p, C.c_int64, C.c_int64, C.POINTER(C.c_double)]
        L.orc_initial_speed.restype = C.c_float
        L.orc_initial_speed.argtypes = [_f32p]
        L.orc_fnv1a.restype = C.c_uint64
        L.orc_fnv1a.argtypes = [C.c_void_p, C.c_int64]
        L.orc_kv_footprint_bytes.restype = C.c_int64
        L.orc_kv_footprint_bytes.argtypes = [C.c_int64] * 5
        self.L = L

    # -- weights -----------------------------------------------------------
    def stream_offset(self, cfg: Cfg) -> int:
        return int(self.L.orc_action_stream_offset(C.byref(cfg)))

    def param_count(self, cfg: Cfg) -> int:
        return int(self.L.orc_action_param_count(C.byref(cfg)))

    def weights(self, cfg: Cfg) -> "PortWeights":
        return PortWeights(self, cfg)

    # -- inputs ------------------------------------------------------------
    def noise(self, seed: int, stride: int, n: int, lane0: int = 0, steps: int = 64) -> np.ndarray:
        out = np.empty((n, steps, 2), np.float32)
        self.L.orc_noise(seed, stride, lane0, n, steps, _fp(out))
        return out

    def synthetic_prefix(self, seed: int, blocks: int, r: int, kv: int) -> np.ndarray:
        out = np.empty((blocks, 2, r, kv), np.float32)
        self.L.orc_synthetic_prefix(seed, blocks, r, kv, _fp(out))
        return out

    def sinusoid(self, positions: int, dim: int) -> np.ndarray:
        out = np.empty((positions, dim), np.float32)
        self.L.orc_sinusoidal_table(positions, dim, _fp(out))
        return out

    # -- the path ----------------------------------------------------------
    def refine(self, cfg: Cfg, w: "PortWeights", prefix: np.ndarray, actions: np.ndarray,
               iters: int | None = None, lane_prefix: np.ndarray | None = None,
               threads: int = 0) -> np.ndarray:
        prefix = np.ascontiguousarray(prefix, np.float32)
        acts = np.array(actions, np.float32, copy=True, order="C")
        n = acts.shape[0]
        r = prefix.shape[-2]
        lp = None
        if lane_prefix is not None:
            lane_prefix = np.ascontiguousarray(lane_prefix, np.int32)
            lp = lane_prefix.ctypes.data_as(_i32p)
        rc = self.L.orc_diffusion_refine(C.byref(cfg), C.byref(w.w), _fp(prefix), r, lp, n,
                                         cfg.diffusion_iters if iters is None else iters,
                                         _fp(acts), threads)
        if rc:
            raise RuntimeError(f"orc_diffusion_refine failed ({rc})")
        return acts

    def rollout(self, actions: np.ndarray, v0: float) -> np.ndarray:
        actions = np.ascontiguousarray(actions, np.float32)
        n, steps = actions.shape[0], actions.shape[1]
        out = np.empty((n, steps, 3), np.float32)
        rc = self.L.orc_rollout(_fp(actions), n, steps, v0, _fp(out))
        if rc:
            raise ValueError("actions_to_trajectory: invalid input (InternalError)")
        return out

    def min_ade(self, traj: np.ndarray, gt: np.ndarray) -> float:
        t = np.ascontiguousarray(traj, np.float32)
        g = np.ascontiguousarray(gt, np.float32)
        out = C.c_double()
        if self.L.orc_min_ade(_fp(t), t.shape[0], t.shape[1], _fp(g), C.byref(out)):
            raise ValueError("min_ade: no samples (InternalError)")
        return out.value

    def diversity(self, traj: np.ndarray) -> float:
        t = np.ascontiguousarray(traj, np.float32)
        out = C.c_double()
        if self.L.orc_diversity(_fp(t), t.shape[0], t.shape[1], C.byref(out)):
            raise ValueError("diversity: need at least 2 samples (InternalError)")
        return out.value

    def initial_speed(self, history: np.ndarray) -> float:
        h = np.ascontiguousarray(history, np.float32)
        return float(self.L.orc_initial_speed(_fp(h)))

    def fnv1a(self, arr: np.ndarray) -> int:
        a = np.ascontiguousarray(arr)
        return int(self.L.orc_fnv1a(a.ctypes.data, a.nbytes))

    def footprint(self, blocks, batch, tokens, kv, eb) -> int:
        return int(self.L.orc_kv_footprint_bytes(blocks, batch, tokens, kv, eb))


class PortWeights:
    def __init__(self, port: Port, cfg: Cfg):
        self.port = port
        self.w = _Weights()
        if port.L.orc_weights_build(C.byref(cfg), C.byref(self.w)):
            raise MemoryError("orc_weights_build failed")
        self.cfg = cfg

    def arena(self) -> np.ndarray:
        """A copy of the whole arena in draw order (safe after this object dies)."""
        return np.ctypeslib.as_array(self.w.arena, shape=(self.w.count,)).copy()

    def tensor(self, which: str, blk: int | None = None):
        """('w' [in][out], 'b' [out]) numpy views of one linear."""
        if blk is None:
            lin = getattr(self.w, which)
        else:
            idx = ["q", "k", "v", "o", "mlp1", "mlp2"].index(which)
            lin = self.w.blocks[blk * 6 + idx]
        w = np.ctypeslib.as_array(lin.w, shape=(lin.in_, lin.out))
        b = np.ctypeslib.as_array(lin.b, shape=(lin.out,))
        return w, b

    def __del__(self):
        try:
            self.port.L.orc_weights_free(C.byref(self.w))
        except Exception:
            pass


class Ref:
    """The reference itself (oracle/_ref/libminivla_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (make -C oracle with /root/reference present)")
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_scenario_prefix.argtypes = [C.POINTER(Cfg), C.c_char_p, C.c_uint64, C.c_int,
                                          C.c_int64, C.c_int, _f32p, C.c_int64,
                                          C.POINTER(C.c_int64), C.POINTER(C.c_uint64), _f32p]
        L.ref_action_generation.argtypes = [C.POINTER(Cfg), _f32p, C.c_int64, C.c_int64,
                                            C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                            C.c_int, _f32p, C.POINTER(C.c_double),
                                            C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        L.ref_rollout.argtypes = [_f32p, C.c_int64, C.c_float, _f32p]
        _i64p = C.POINTER(C.c_int64)
        L.ref_reasoning_io.argtypes = [C.POINTER(Cfg), C.c_char_p, C.c_uint64, C.c_int, _f32p, C.c_int64,
                                       _i64p, _i64p, C.c_int64, _i64p, _i64p, C.c_int64, _i64p, _i64p]
        L.ref_action_weights.argtypes = [C.POINTER(Cfg), C.c_int, _f32p, C.c_int64,
                                         C.POINTER(C.c_int64)]
        L.ref_parse_latency_report.argtypes = [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        L.ref_min_ade.argtypes = [_f32p, C.c_int64, C.c_int64, _f32p, C.POINTER(C.c_double)]
        L.ref_diversity.argtypes = [_f32p, C.c_int64, C.c_int64, C.POINTER(C.c_double)]
        self.L = L

    def _check(self, rc):
        if rc:
            raise RuntimeError(f"reference error {rc}: {self.L.ref_last_error().decode()}")

    def scenario_prefix(self, cfg: Cfg, scenario: str, sampler_seed=1, stochastic=True,
                        forced_cot=0, static_kv=True):
        r = C.c_int64()
        fp = C.c_uint64()
        v0 = C.c_float()
        self._check(self.L.ref_scenario_prefix(C.byref(cfg), scenario.encode(), sampler_seed,
                                               int(stochastic), forced_cot, int(static_kv),
                                               None, 0, C.byref(r), C.byref(fp), C.byref(v0)))
        out = np.empty((cfg.decoder_blocks, 2, r.value, cfg.kv_dim), np.float32)
        self._check(self.L.ref_scenario_prefix(C.byref(cfg), scenario.encode(), sampler_seed,
                                               int(stochastic), forced_cot, int(static_kv),
                                               _fp(out), out.size, C.byref(r), C.byref(fp),
                                               C.byref(v0)))
        return out, int(fp.value), float(v0.value)

    def action_generation(self, cfg: Cfg, prefix: np.ndarray, n: int, seed=2, stride=1,
                          static_kv=True, graph=True, single=True, parallel=True):
        prefix = np.ascontiguousarray(prefix, np.float32)
        r = prefix.shape[-2]
        out = np.empty((n, cfg.action_steps, 2), np.float32)
        ms = C.c_double()
        kvb = C.c_int64()
        it = C.c_double()
        self._check(self.L.ref_action_generation(C.byref(cfg), _fp(prefix), r, n, seed, stride,
                                                 int(static_kv), int(graph), int(single),
                                                 int(parallel), _fp(out), C.byref(ms),
                                                 C.byref(kvb), C.byref(it)))
        self.last_iter_ms = float(it.value)  # sum of DiffusionResult::iter_ms
        return out, float(ms.value), int(kvb.value)

    def reasoning_io(self, cfg: Cfg, scenario: str, sampler_seed=1, stochastic=True):
        """(vision rows [P][hidden], prompt ids, decode-loop ids, T, m) of the
        reference's reasoning stage on a scenario (ref_reasoning_io)."""
        i64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))
        P, npr, m, T = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self.L.ref_reasoning_io(C.byref(cfg), scenario.encode(), sampler_seed, int(stochastic),
                                            None, 0, C.byref(P), None, 0, C.byref(npr), None, 0,
                                            C.byref(m), C.byref(T)))
        vis = np.empty((P.value, cfg.hidden_dim), np.float32)
        prompt = np.empty(npr.value, np.int64)
        ids = np.empty(max(m.value, 1), np.int64)
        self._check(self.L.ref_reasoning_io(C.byref(cfg), scenario.encode(), sampler_seed, int(stochastic),
                                            _fp(vis), vis.size, C.byref(P), i64(prompt), prompt.size,
                                            C.byref(npr), i64(ids), ids.size, C.byref(m), C.byref(T)))
        return vis, prompt, ids[: m.value], int(T.value), int(m.value)

    def rollout(self, actions: np.ndarray, v0: float) -> np.ndarray:
        actions = np.ascontiguousarray(actions, np.float32)
        n = actions.shape[0]
        out = np.empty((n, 64, 3), np.float32)
        self._check(self.L.ref_rollout(_fp(actions), n, v0, _fp(out)))
        return out

    def parse_latency_report(self, doc: str) -> tuple[int, float]:
        """LatencyReport::from_json of the reference (profiler.cpp:49-66)."""
        n = C.c_int64()
        ms = C.c_double()
        self._check(self.L.ref_parse_latency_report(doc.encode(), C.byref(n), C.byref(ms)))
        return n.value, ms.value

    def min_ade(self, traj: np.ndarray, gt: np.ndarray) -> float:
        t = np.ascontiguousarray(traj, np.float32)
        g = np.ascontiguousarray(gt, np.float32)
        out = C.c_double()
        self._check(self.L.ref_min_ade(_fp(t), t.shape[0], t.shape[1], _fp(g), C.byref(out)))
        return out.value

    def diversity(self, traj: np.ndarray) -> float:
        t = np.ascontiguousarray(traj, np.float32)
        out = C.c_double()
        self._check(self.L.ref_diversity(_fp(t), t.shape[0], t.shape[1], C.byref(out)))
        return out.value

    def action_weight(self, cfg: Cfg, which: int) -> np.ndarray:
        cnt = C.c_int64()
        self._check(self.L.ref_action_weights(C.byref(cfg), which, None, 0, C.byref(cnt)))
        out = np.empty(cnt.value, np.float32)
        self._check(self.L.ref_action_weights(C.byref(cfg), which, _fp(out), out.size,
                                              C.byref(cnt)))
        return out


def have_ref() -> bool:
    return os.path.exists(REF_SO)
