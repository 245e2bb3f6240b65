"""B200-native single-reasoning diffusion action generation (arXiv 2605.08975).

Python mirror of the reference's action-generation interface
(``Engine::run_action_generation``, /root/reference/proj/include/minivla/
pipeline.hpp:145-148) over the C-ABI library ``libalpa_action.so``
(include/alpa_action.h).  All compute runs in hand-written sm_100a kernels;
there is no CPU fallback: importing this package without the built library,
or running it without a Blackwell GPU, raises.

    cfg = ModelConfig(action_hidden_dim=2048, kv_dim=1024, heads=8,
                      decoder_blocks=36, dtype="bf16")
    gen = ActionGenerator(cfg)                 # weights drawn on device
    gen.bind_prefix_synthetic(seed=4242, r=2048)
    res = gen.run_action_generation(InferenceRequest(num_trajectories=6))
    res.actions   # [6][64][2] f32   (accel, curvature)
    res.trajectories  # [6][64][3] f32 (x, y, yaw)
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ALPA_LIB") or os.path.join(_HERE, "libalpa_action.so")

ALPA_OK, ALPA_ERR_IO, ALPA_ERR_CONFIG, ALPA_ERR_INTERNAL = 0, 1, 2, 3
DTYPES = {"f32": 0, "fp32": 0, "float32": 0, "bf16": 1, "bfloat16": 1}
KV_STRATEGIES = {"dynamic": 0, "static": 1}
EXECUTORS = {"eager": 0, "graph": 1}
TOPOLOGIES = {"multi": 0, "single": 1}


class Error(RuntimeError):
    """minivla::Error (common.hpp:12-14)."""

    code = ALPA_ERR_INTERNAL


class IoError(Error):
    code = ALPA_ERR_IO


class ConfigError(Error):
    code = ALPA_ERR_CONFIG


class InternalError(Error):
    code = ALPA_ERR_INTERNAL


_ERRORS = {ALPA_ERR_IO: IoError, ALPA_ERR_CONFIG: ConfigError, ALPA_ERR_INTERNAL: InternalError}


class _Cfg(C.Structure):
    _fields_ = [
        ("vision_blocks", C.c_int64), ("decoder_blocks", C.c_int64), ("hidden_dim", C.c_int64),
        ("action_hidden_dim", C.c_int64), ("kv_dim", C.c_int64), ("heads", C.c_int64),
        ("vocab_size", C.c_int64), ("patch_size", C.c_int64), ("action_steps", C.c_int64),
        ("diffusion_iters", C.c_int64), ("update_scale", C.c_float), ("dtype", C.c_int32),
        ("weight_seed", C.c_uint64),
    ]


class _Req(C.Structure):
    _fields_ = [
        ("num_trajectories", C.c_int64), ("lane0", C.c_int64), ("action_init_seed", C.c_uint64),
        ("action_seed_stride", C.c_uint64), ("diffusion_iters", C.c_int64),
        ("topology", C.c_int32), ("kv_strategy", C.c_int32), ("executor", C.c_int32),
        ("v0", C.c_float),
    ]


class Stats(C.Structure):
    """alpa_stats: device time, kernel / graph launch counts, kv footprint."""

    _fields_ = [
        ("device_ms", C.c_double), ("kernel_launches", C.c_int64), ("graph_launches", C.c_int64),
        ("graph_nodes", C.c_int64), ("kv_bytes", C.c_int64), ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64), ("n_iter", C.c_int64), ("iter_ms", C.c_double * 64),
        ("bytes_allocated", C.c_int64),
    ]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "iter_ms"}
        d["iter_ms"] = [self.iter_ms[i] for i in range(min(self.n_iter, 64))]
        return d


class KernelProf(C.Structure):
    _fields_ = [("name", C.c_char * 40), ("launches", C.c_int64), ("total_ms", C.c_double),
                ("flops", C.c_double), ("bytes", C.c_double)]


_f32p = C.POINTER(C.c_float)
_lib = None


def lib():
    """The loaded C-ABI library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.alpa_version.restype = C.c_char_p
        L.alpa_last_error.restype = C.c_char_p
        L.alpa_last_error.argtypes = [C.c_void_p]
        L.alpa_ctx_create.argtypes = [P(_Cfg), C.c_int, P(C.c_void_p)]
        L.alpa_ctx_destroy.argtypes = [C.c_void_p]
        L.alpa_set_stream.argtypes = [C.c_void_p, C.c_void_p]
        L.alpa_default_cfg.argtypes = [P(_Cfg)]
        L.alpa_validate_cfg.argtypes = [P(_Cfg)]
        L.alpa_load_weights_seeded.argtypes = [C.c_void_p, C.c_uint64, C.c_int64]
        L.alpa_load_weights_host.argtypes = [C.c_void_p, _f32p, C.c_int64]
        L.alpa_weight_stream_offset.restype = C.c_int64
        L.alpa_weight_stream_offset.argtypes = [P(_Cfg)]
        L.alpa_action_param_count.restype = C.c_int64
        L.alpa_action_param_count.argtypes = [P(_Cfg)]
        L.alpa_bind_prefix.argtypes = [C.c_void_p, _f32p, C.c_int64, C.c_int64]
        L.alpa_bind_prefix_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64]
        L.alpa_bind_prefix_synthetic.argtypes = [C.c_void_p, C.c_uint64, C.c_int64]
        L.alpa_synthesize_prefix.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int64]
        L.alpa_prefix_device.argtypes = [C.c_void_p, P(C.c_void_p), P(C.c_int64)]
        L.alpa_set_lane_prefix.argtypes = [C.c_void_p, P(C.c_int32), C.c_int64]
        L.alpa_generate.argtypes = [C.c_void_p, P(_Req), _f32p, _f32p, P(Stats)]
        L.alpa_generate_device.argtypes = [C.c_void_p, P(_Req), C.c_void_p, C.c_void_p,
                                           C.c_void_p, P(Stats)]
        L.alpa_profile.argtypes = [C.c_void_p, P(_Req), C.c_int64, P(KernelProf), C.c_int32,
                                   P(C.c_int32)]
        L.alpa_host_noise.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, C.c_int64,
                                      _f32p]
        L.alpa_initial_speed.restype = C.c_float
        L.alpa_initial_speed.argtypes = [_f32p]
        L.alpa_rollout.argtypes = [C.c_void_p, _f32p, C.c_int64, C.c_float, _f32p]
        L.alpa_kv_footprint_bytes.restype = C.c_int64
        L.alpa_kv_footprint_bytes.argtypes = [C.c_int64] * 5
        _f64p = C.POINTER(C.c_double)
        L.alpa_eval_open_loop.argtypes = [C.c_void_p, _f32p, _f32p, C.c_int64, C.c_int64, C.c_int64,
                                          _f64p, _f64p]
        L.alpa_eval_open_loop_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                                 C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        _i64p = C.POINTER(C.c_int64)
        L.alpa_reasoning_begin.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
        L.alpa_reasoning_prefill.argtypes = [C.c_void_p, _f32p, C.c_int64, _i64p, C.c_int64, _f32p]
        L.alpa_reasoning_decode.argtypes = [C.c_void_p, _i64p, _f32p]
        L.alpa_reasoning_seal.argtypes = [C.c_void_p, _i64p]
        L.alpa_sample_token.argtypes = [_f32p, C.c_int64, C.c_int, C.POINTER(C.c_uint64), _i64p]
        _lib = L
    return _lib


def sample_token(logits: np.ndarray, stochastic: bool, state: int) -> tuple[int, int]:
    """minivla::sample_token (model.cpp:30-54), host, bit-exact: returns
    (token, advanced Rng state)."""
    lg = np.ascontiguousarray(logits, np.float32)
    st = C.c_uint64(state)
    tok = C.c_int64()
    _check(lib().alpa_sample_token(_fp(lg), lg.size, int(stochastic), C.byref(st), C.byref(tok)))
    return int(tok.value), int(st.value)


def _check(rc: int, ctx=None) -> None:
    if rc != ALPA_OK:
        msg = lib().alpa_last_error(ctx).decode()
        raise _ERRORS.get(rc, InternalError)(msg)


def _fp(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(_f32p)


@dataclasses.dataclass
class ModelConfig:
    """ModelConfig (model.hpp:12-29) + the compute dtype of this build."""

    vision_blocks: int = 4
    decoder_blocks: int = 6
    hidden_dim: int = 64
    action_hidden_dim: int = 32
    kv_dim: int = 32
    heads: int = 4
    vocab_size: int = 512
    patch_size: int = 14
    action_steps: int = 64
    diffusion_iters: int = 10
    update_scale: float = 0.1
    max_new_tokens: int = 256  # reasoning-side field, kept for parity of the struct
    weight_seed: int = 1234
    dtype: str = "f32"

    def head_dim(self) -> int:
        return self.kv_dim // self.heads

    def _c(self) -> _Cfg:
        return _Cfg(self.vision_blocks, self.decoder_blocks, self.hidden_dim,
                    self.action_hidden_dim, self.kv_dim, self.heads, self.vocab_size,
                    self.patch_size, self.action_steps, self.diffusion_iters, self.update_scale,
                    DTYPES[self.dtype], self.weight_seed)

    def validate(self) -> None:
        """ModelConfig::validate (model.cpp:9-24); raises ConfigError."""
        _check(lib().alpa_validate_cfg(C.byref(self._c())))

    def weight_stream_offset(self) -> int:
        return int(lib().alpa_weight_stream_offset(C.byref(self._c())))

    def action_param_count(self) -> int:
        return int(lib().alpa_action_param_count(C.byref(self._c())))


@dataclasses.dataclass
class InferenceRequest:
    """The InferenceRequest fields the path consumes (pipeline.hpp:97-113)."""

    num_trajectories: int = 1
    topology: str = "single"
    kv_strategy: str = "static"
    executor: str = "graph"
    action_init_seed: int = 2
    action_seed_stride: int = 1
    v0: float = 5.0            # initial_speed_from_history(pose_history)
    lane0: int = 0             # global lane offset (multi-GPU slices)
    diffusion_iters: int = 0   # 0 -> ModelConfig.diffusion_iters

    def _c(self) -> _Req:
        return _Req(self.num_trajectories, self.lane0, self.action_init_seed,
                    self.action_seed_stride, self.diffusion_iters, TOPOLOGIES[self.topology],
                    KV_STRATEGIES[self.kv_strategy], EXECUTORS[self.executor], self.v0)


@dataclasses.dataclass
class ActionResult:
    actions: np.ndarray       # [N][64][2] (accel, curvature)   (model.cpp:638-650)
    trajectories: np.ndarray  # [N][64][3] (x, y, yaw)           (pipeline.cpp:124-148)
    stats: dict


class ActionGenerator:
    """One device context: action-expert weights + the single prefix copy +
    the captured K-loop graph.  Mirrors Engine's action-generation half
    (pipeline.hpp:130-165).  Not thread-safe (one logical stream)."""

    def __init__(self, cfg: ModelConfig, device: int = 0, weights: str | np.ndarray = "seeded",
                 stream_offset: int = -1):
        self.cfg = cfg
        self._h = C.c_void_p()
        _check(lib().alpa_ctx_create(C.byref(cfg._c()), device, C.byref(self._h)))
        if isinstance(weights, np.ndarray):
            arena = np.ascontiguousarray(weights, np.float32)
            _check(lib().alpa_load_weights_host(self._h, _fp(arena), arena.size), self._h)
        else:
            _check(lib().alpa_load_weights_seeded(self._h, cfg.weight_seed, stream_offset),
                   self._h)

    def close(self) -> None:
        if self._h:
            lib().alpa_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- prefix ------------------------------------------------------------
    def bind_prefix(self, kv: np.ndarray) -> None:
        """Host f32 prefix [B][2][r][kv] (single) or [n][B][2][r][kv] (multi)."""
        kv = np.ascontiguousarray(kv, np.float32)
        n = 1 if kv.ndim == 4 else kv.shape[0]
        _check(lib().alpa_bind_prefix(self._h, _fp(kv), n, kv.shape[-2]), self._h)

    def bind_prefix_synthetic(self, seed: int, r: int) -> None:
        _check(lib().alpa_bind_prefix_synthetic(self._h, seed, r), self._h)

    def bind_prefix_device(self, ptr: int, n_prefix: int, r: int) -> None:
        _check(lib().alpa_bind_prefix_device(self._h, C.c_void_p(ptr), n_prefix, r), self._h)

    def synthesize_prefix(self, dst_ptr: int, seed: int, r: int) -> None:
        """Write the synthetic scene prefix into a caller device buffer (on the
        ctx stream)."""
        _check(lib().alpa_synthesize_prefix(self._h, C.c_void_p(dst_ptr), seed, r), self._h)

    def prefix_bytes(self, r: int, n_prefix: int = 1) -> int:
        es = 2 if DTYPES[self.cfg.dtype] == 1 else 4
        return n_prefix * self.cfg.decoder_blocks * 2 * r * self.cfg.kv_dim * es

    def prefix_device(self) -> tuple[int, int]:
        p, nb = C.c_void_p(), C.c_int64()
        _check(lib().alpa_prefix_device(self._h, C.byref(p), C.byref(nb)), self._h)
        return int(p.value or 0), int(nb.value)

    def set_lane_prefix(self, lane_map) -> None:
        m = np.ascontiguousarray(lane_map, np.int32)
        _check(lib().alpa_set_lane_prefix(self._h, m.ctypes.data_as(C.POINTER(C.c_int32)),
                                          m.size), self._h)

    # -- reasoning-stage KV producer ------------------------------
    def reasoning_begin(self, lanes: int, capacity: int) -> None:
        """Static in-place KV of `capacity` tokens per lane (T + max_new_tokens,
        pipeline.cpp:281-286) in the action stage's prefix layout."""
        _check(lib().alpa_reasoning_begin(self._h, lanes, capacity), self._h)

    def reasoning_prefill(self, vision: np.ndarray, prompt_ids, lanes: int = 1) -> np.ndarray:
        """Model::prefill over [vision rows | prompt embeddings] + positions;
        vision [P][h] (shared by every lane) or [lanes][P][h]. Returns logits
        [lanes][vocab]."""
        v = np.ascontiguousarray(vision, np.float32)
        if v.ndim == 2:
            v = np.ascontiguousarray(np.broadcast_to(v, (lanes,) + v.shape))
        ids = np.ascontiguousarray(prompt_ids, np.int64)
        out = np.empty((v.shape[0], self.cfg.vocab_size), np.float32)
        _check(lib().alpa_reasoning_prefill(self._h, _fp(v), v.shape[1],
                                            ids.ctypes.data_as(C.POINTER(C.c_int64)), ids.size,
                                            _fp(out)), self._h)
        return out

    def reasoning_decode(self, ids) -> np.ndarray:
        """One decode step: ids [lanes] at the next position. Returns logits."""
        t = np.ascontiguousarray(ids, np.int64)
        out = np.empty((t.size, self.cfg.vocab_size), np.float32)
        _check(lib().alpa_reasoning_decode(self._h, t.ctypes.data_as(C.POINTER(C.c_int64)), _fp(out)),
               self._h)
        return out

    def reasoning_seal(self) -> int:
        """KvCache::seal_reasoning: the produced KV becomes the action prefix in place."""
        r = C.c_int64()
        _check(lib().alpa_reasoning_seal(self._h, C.byref(r)), self._h)
        return int(r.value)

    def run_reasoning(self, vision: np.ndarray, prompt_ids, lanes: int = 1, max_new_tokens: int = 256,
                      sampler_seed: int = 1, stochastic: bool = True, forced_cot_tokens: int = 0,
                      termination_token: int = 0, forced_ids=None) -> dict:
        """Engine::reasoning_pass (pipeline.cpp:279-390) around the device
        producer: prefill, then the decode loop with the reference's host
        sampler (per-lane Rng(sampler_seed + lane)), then seal.  forced_ids
        [m][lanes] teacher-forces the fed-back ids instead of sampling.
        Returns {cot_tokens, token_count, r, prompt_tokens}."""
        v = np.asarray(vision, np.float32)
        T = v.shape[-2] + len(prompt_ids)
        self.reasoning_begin(lanes, T + max_new_tokens)
        logits = self.reasoning_prefill(v, prompt_ids, lanes)
        states = [sampler_seed + l for l in range(lanes)]
        done = [False] * lanes
        cot = [[] for _ in range(lanes)]
        forced = forced_cot_tokens > 0
        max_m = min(forced_cot_tokens, max_new_tokens) if forced else max_new_tokens
        m = 0
        while m < max_m:
            if all(done) and not forced:
                break
            if forced_ids is not None:
                if m >= len(forced_ids):
                    break
                ids = [int(x) for x in np.atleast_1d(forced_ids[m])]
            else:
                ids = []
                for l in range(lanes):
                    tok, states[l] = sample_token(logits[l], stochastic, states[l])
                    ids.append(tok)
            for l in range(lanes):
                if not done[l]:
                    if not forced and ids[l] == termination_token:
                        done[l] = True
                    else:
                        cot[l].append(ids[l])
            m += 1
            logits = self.reasoning_decode(ids)
        r = self.reasoning_seal()
        return {"cot_tokens": cot, "token_count": m, "r": r, "prompt_tokens": T}

    def set_stream(self, stream_handle: int) -> None:
        _check(lib().alpa_set_stream(self._h, C.c_void_p(stream_handle)), self._h)

    # -- the path ----------------------------------------------------------
    def run_action_generation(self, req: InferenceRequest) -> ActionResult:
        """Engine::run_action_generation + actions_to_trajectory: host in, host out."""
        n = req.num_trajectories
        acts = np.empty((max(n, 0), self.cfg.action_steps, 2), np.float32)
        traj = np.empty((max(n, 0), self.cfg.action_steps, 3), np.float32)
        st = Stats()
        _check(lib().alpa_generate(self._h, C.byref(req._c()), _fp(acts), _fp(traj),
                                   C.byref(st)), self._h)
        return ActionResult(acts, traj, st.as_dict())

    def generate_device(self, req: InferenceRequest, d_noise: int, d_actions: int,
                        d_traj: int = 0, stats: bool = False) -> dict | None:
        """Device-resident variant: pointers to HBM buffers (e.g. torch data_ptr())."""
        st = Stats() if stats else None
        _check(lib().alpa_generate_device(self._h, C.byref(req._c()), C.c_void_p(d_noise),
                                          C.c_void_p(d_actions), C.c_void_p(d_traj or None),
                                          C.byref(st) if st is not None else None), self._h)
        return st.as_dict() if st is not None else None

    def profile(self, req: InferenceRequest, iters: int = 1) -> list[dict]:
        """Per-kernel CUDA-event times of `iters` eager iterations (+ rollout)."""
        buf = (KernelProf * 64)()
        n = C.c_int32()
        _check(lib().alpa_profile(self._h, C.byref(req._c()), iters, buf, 64, C.byref(n)),
               self._h)
        return [dict(name=buf[i].name.decode(), launches=buf[i].launches,
                     total_ms=buf[i].total_ms, flops=buf[i].flops, bytes=buf[i].bytes)
                for i in range(n.value)]

    def eval_open_loop(self, traj: np.ndarray, gt: np.ndarray | None = None,
                       diversity: bool = True) -> tuple[np.ndarray, np.ndarray | None]:
        """minivla::min_ade / minivla::diversity (eval.cpp:39-59) of a batch of scenes on
        the device, bit-exact: traj [scenes][n][steps][3] (or [n][steps][3]), gt
        [scenes][steps][3] (or [steps][3]).  Returns (min_ade [scenes], diversity
        [scenes] or None)."""
        t = np.ascontiguousarray(traj, np.float32)
        if t.ndim == 3:
            t = t[None]
        scenes, n, steps = t.shape[0], t.shape[1], t.shape[2]
        g = None
        if gt is not None:
            g = np.ascontiguousarray(gt, np.float32).reshape(scenes, steps, 3)
        ade = np.empty(scenes, np.float64)
        div = np.empty(scenes, np.float64) if diversity else None
        f64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None  # noqa: E731
        _check(lib().alpa_eval_open_loop(self._h, _fp(t), _fp(g) if g is not None else None, scenes,
                                         n, steps, f64(ade) if g is not None else None, f64(div)),
               self._h)
        return (ade if g is not None else None), div

    def rollout(self, actions: np.ndarray, v0: float) -> np.ndarray:
        a = np.ascontiguousarray(actions, np.float32)
        out = np.empty((a.shape[0], a.shape[1], 3), np.float32)
        _check(lib().alpa_rollout(self._h, _fp(a), a.shape[0], v0, _fp(out)), self._h)
        return out


def host_noise(seed: int, stride: int, n: int, lane0: int = 0, steps: int = 64) -> np.ndarray:
    """Rng::normal lane noise (pipeline.cpp:415-424), bit-exact, [n][steps][2]."""
    out = np.empty((n, steps, 2), np.float32)
    lib().alpa_host_noise(seed, stride, lane0, n, steps, _fp(out))
    return out


def initial_speed(history: np.ndarray) -> float:
    """initial_speed_from_history (pipeline.cpp:150-156); history [16][3]."""
    h = np.ascontiguousarray(history, np.float32)
    return float(lib().alpa_initial_speed(_fp(h)))


def kv_footprint_bytes(blocks: int, batch: int, tokens: int, kv_dim: int, elem_bytes: int) -> int:
    return int(lib().alpa_kv_footprint_bytes(blocks, batch, tokens, kv_dim, elem_bytes))


def version() -> str:
    return lib().alpa_version().decode()


def build(verbose: bool = False) -> str:
    """Compile libalpa_action.so in-tree for sm_100a (nvcc cross-compiles
    without a GPU)."""
    import subprocess

    out = subprocess.run(["make", "-C", _HERE, "-j8"], capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"build failed:\n{out.stdout}\n{out.stderr}")
    return LIB_PATH
