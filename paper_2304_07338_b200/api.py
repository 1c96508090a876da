"""Python mirror of the reference's pf:: render-path API over the C ABI.

Reference interface (namespace pf, /root/reference/proj + SPEC.md) -> here:
  pf::Medium(grid, tf, density_scale)        Context.upload_volume + set_medium
  pf::delta_track(medium, ray, rng)          Context.delta_track_batch
  pf::transmittance(medium, a, b, rng, n)    Context.transmittance_batch
  pf::make_rng(seed, stream, index)          Context.rng_doubles (device PCG32)
  pf::trace_photons(medium, lights, cfg)     Context.trace_photons    (photon.hpp:56, Alg. 1)
  render_neural(scene, field, cfg, cam, spp) Context.render_neural
  forward / infer_radiance                   Context.field_query
  build / knn_phase                          Context.knn_build / knn_query
  Eq.6 + Eq.7 target gather, make_batch      Context.knn_targets / make_batch
Errors: ValueError where the reference throws std::invalid_argument,
RuntimeError for std::runtime_error / CUDA failures.

Array arguments may be numpy arrays (host; staged by the library) or CUDA
torch tensors (device; used in place, results stay on the device).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _lib
from ._lib import STREAM, check, lib
from .scene import PHOTON_DTYPE, CameraSpec, validate_tf

# ------------------------------------------------------------ configs -----


@dataclass
class HashGrid:
    dims: int
    levels: int
    features: int
    base_res: int = 4
    growth: float = 2.0
    log2_table: int = 15

    def c(self) -> _lib.HashGridDesc:
        return _lib.HashGridDesc(self.dims, self.levels, self.features, self.base_res,
                                 float(self.growth), self.log2_table)


@dataclass
class FieldConfig:
    """PhotonField = pos hash grid + dir hash grid + MLP."""
    pos: HashGrid = field(default_factory=lambda: HashGrid(3, 8, 4))
    dir: HashGrid = field(default_factory=lambda: HashGrid(2, 8, 4))
    hidden_layers: int = 5
    width: int = 64
    psi: float = 5.0

    @staticmethod
    def desk() -> "FieldConfig":
        """SPEC.md:434 desk scale: 8 levels x 4 features, T = 2^15."""
        return FieldConfig()

    @staticmethod
    def paper() -> "FieldConfig":
        """PAPER.md:351 / SPEC.md:358: 16 levels x 8 features, T = 2^19, growth 2."""
        return FieldConfig(HashGrid(3, 16, 8, 4, 2.0, 19), HashGrid(2, 16, 8, 4, 2.0, 19))

    def c(self) -> _lib.FieldDesc:
        return _lib.FieldDesc(self.pos.c(), self.dir.c(), self.hidden_layers, self.width,
                              float(self.psi))

    def param_count(self) -> int:
        n = C.c_size_t()
        check(lib().pf_field_param_count(C.byref(self.c()), C.byref(n)))
        return n.value

    def init_params(self, seed: int = 0, embed_scale: float = 1e-4,
                    bias_scale: float = 0.0) -> np.ndarray:
        """Deterministic init from make_rng(seed, FieldInit, 0)."""
        out = np.empty(self.param_count(), dtype=np.float32)
        check(lib().pf_field_init(C.byref(self.c()), seed, embed_scale, bias_scale,
                                  out.ctypes.data))
        return out


@dataclass
class RenderConfig:
    spp: int = 1
    g: float = 0.0
    seed: int = 0
    w_d: float = 1.0
    w_i: float = 1.0
    background: tuple = (0.0, 0.0, 0.0)
    mode: str = "fast"            # "parity" (binary64, delta-trial NEE) | "fast"
    nee_trials: int = 1
    use_field: bool = True
    tile: tuple = (16, 16)
    shard_index: int = 0
    shard_count: int = 1

    def c(self) -> _lib.RenderDesc:
        mode = {"parity": _lib.PF_MODE_PARITY, "fast": _lib.PF_MODE_FAST}[self.mode]
        return _lib.RenderDesc(self.spp, float(self.g), self.seed, float(self.w_d),
                               float(self.w_i), (C.c_double * 3)(*self.background), mode,
                               self.nee_trials, int(self.use_field), self.tile[0], self.tile[1],
                               self.shard_index, self.shard_count)


@dataclass
class PathTraceConfig:
    """render_path_traced's path controls (roulette as in
    trace_photons, photon.hpp:29-37)."""
    max_bounces: int = 16
    rr_start_bounce: int = 3
    rr_min_survival: float = 0.05
    rr_max_survival: float = 0.95

    def c(self) -> _lib.PathDesc:
        return _lib.PathDesc(self.max_bounces, self.rr_start_bounce, float(self.rr_min_survival),
                             float(self.rr_max_survival))


@dataclass
class TraceConfig:
    """pf::TraceConfig (proj/include/pf/photon.hpp:29-37)."""
    n_total: int = 100000
    phase_set: list = field(default_factory=lambda: [-0.75, 0.0, 0.75])
    max_bounces: int = 16
    rr_start_bounce: int = 3
    rr_min_survival: float = 0.05
    rr_max_survival: float = 0.95
    seed: int = 0


@dataclass
class AdamConfig:
    """AdamState + the rMSE epsilon of train_step."""
    lr: float = 9e-4
    beta1: float = 0.9
    beta2: float = 0.99
    eps: float = 1e-8
    decay: float = 0.92
    decay_start: float = 0.7
    decay_interval: int = 25
    eps_rel: float = 0.01

    def c(self) -> _lib.AdamDesc:
        return _lib.AdamDesc(self.lr, self.beta1, self.beta2, self.eps, self.decay, self.decay_start,
                             int(self.decay_interval), self.eps_rel)


@dataclass
class TrainConfig:
    """TrainConfig + KnnSchedule; default = the paper's 1M-row
    four-step staggered schedule (PAPER.md table tab:training_target_radii)."""
    total_steps: int = 3000
    batch_size: int = 1 << 16
    K: int = 1024
    schedule_ends: tuple = (0.36, 0.63, 0.90, 1.0)
    schedule_radii: tuple = (0.25, 0.50, 2.50, 5.0)
    psi: float = 5.0
    seed: int = 0


@dataclass
class TrainResult:
    loss_history: np.ndarray
    knn_ms: float       # cumulative make_batch (KNN + Eq. 6/7) device time
    step_ms: float      # cumulative train_step device time
    knn_ms_steps: np.ndarray = None
    step_ms_steps: np.ndarray = None
    radius: np.ndarray = None
    lr: np.ndarray = None
    first_step: int = 0  # absolute step of entry 0 (a resumed run starts at its checkpoint)

    def write_log(self, path) -> None:
        """Training log, one line per step: step, loss, radius, lr,
        cumulative knn_time (ms), as comma-separated text."""
        cum = np.cumsum(self.knn_ms_steps)
        with open(path, "w") as f:
            f.write("step,loss,radius,lr,knn_time_ms\n")
            for i, l in enumerate(self.loss_history):
                f.write(f"{self.first_step + i},{l:.17g},{self.radius[i]:.17g},{self.lr[i]:.17g},{cum[i]:.6f}\n")


def lr_at(step: int, total: int, adam: "AdamConfig | None" = None) -> float:
    """lr(step) = lr0 * decay^floor(max(0, step - decay_start * total) / interval)."""
    a = adam or AdamConfig()
    import math
    return a.lr * a.decay ** math.floor(max(0.0, step - a.decay_start * total) / a.decay_interval)


_CKPT_MAGIC = b"PFFC"


def save_checkpoint(path, cfg: "FieldConfig", phase_set, step: int, params, m, v,
                    adam: "AdamConfig | None" = None, total_steps: int = 0) -> None:
    """Field checkpoint: header (configs, psi, G, next step, the
    Adam hyperparameters and the run's total_steps -- everything train() needs
    to continue at `step`), then the flat parameter vector and both Adam
    moments, little-endian binary64.  Version 2 (version 1 had no Adam block)."""
    import struct
    gs = np.asarray(phase_set, np.float64)
    a = adam or AdamConfig()
    with open(path, "wb") as f:
        f.write(_CKPT_MAGIC + struct.pack("<I", 2))
        for hg in (cfg.pos, cfg.dir):
            f.write(struct.pack("<iiiidi", hg.dims, hg.levels, hg.features, hg.base_res, float(hg.growth),
                                hg.log2_table))
        f.write(struct.pack("<iid", cfg.hidden_layers, cfg.width, float(cfg.psi)))
        f.write(struct.pack("<I", len(gs)) + gs.astype("<f8").tobytes())
        f.write(struct.pack(_CKPT_ADAM, a.lr, a.beta1, a.beta2, a.eps, a.decay, a.decay_start, a.eps_rel,
                            int(a.decay_interval), int(total_steps)))
        f.write(struct.pack("<QQ", int(step), len(params)))
        for arr in (params, m, v):
            f.write(np.asarray(arr, np.float64).astype("<f8").tobytes())


_CKPT_ADAM = "<7diQ"


def _parse_checkpoint(path):
    import struct
    with open(path, "rb") as f:
        buf = f.read()
    if buf[:4] != _CKPT_MAGIC:
        raise ValueError("field checkpoint: bad magic")
    (ver,) = struct.unpack_from("<I", buf, 4)
    if ver not in (1, 2):
        raise ValueError(f"field checkpoint: unsupported version {ver}")
    o = 8
    grids = []
    for _ in range(2):
        d, lv, fe, br, gr, lt = struct.unpack_from("<iiiidi", buf, o)
        o += struct.calcsize("<iiiidi")
        grids.append(HashGrid(d, lv, fe, br, gr, lt))
    hl, wd, psi = struct.unpack_from("<iid", buf, o)
    o += struct.calcsize("<iid")
    (ng,) = struct.unpack_from("<I", buf, o)
    o += 4
    gs = np.frombuffer(buf, "<f8", ng, o).copy()
    o += 8 * ng
    adam, total = None, 0
    if ver == 2:
        lr, b1, b2, eps, dec, dstart, erel, dint, total = struct.unpack_from(_CKPT_ADAM, buf, o)
        o += struct.calcsize(_CKPT_ADAM)
        adam = AdamConfig(lr, b1, b2, eps, dec, dstart, dint, erel)
    step, n = struct.unpack_from("<QQ", buf, o)
    o += 16
    arrs = [np.frombuffer(buf, "<f8", n, o + 8 * n * k).copy() for k in range(3)]
    if o + 24 * n != len(buf):
        raise ValueError("field checkpoint: truncated or oversized")
    cfg = FieldConfig(pos=grids[0], dir=grids[1], hidden_layers=hl, width=wd, psi=psi)
    return cfg, list(gs), step, arrs, adam, total


def load_checkpoint(path):
    """-> (FieldConfig, phase_set, next step, params, m, v) (binary64 arrays)."""
    cfg, gs, step, arrs, _, _ = _parse_checkpoint(path)
    return cfg, gs, step, *arrs


def checkpoint_training_state(path):
    """-> (AdamConfig or None for a version-1 file, total_steps (0 = unknown))."""
    _, _, _, _, adam, total = _parse_checkpoint(path)
    return adam, total


@dataclass
class TraceResult:
    """pf::TraceResult (photon.hpp:39-46)."""
    photons: Any                 # PHOTON_DTYPE array (host) or uint8 CUDA tensor [n, 40]
    phase_set: list
    emitted_per_pair: np.ndarray  # index = light * |G| + phase
    n_lights: int


# ------------------------------------------------------------- helpers ----


def _is_torch(x: Any) -> bool:
    return type(x).__module__.startswith("torch")


def _in(x: Any, dtype, shape_tail=None) -> tuple[int, Any]:
    """(pointer, keepalive) for an input array."""
    if _is_torch(x):
        if not x.is_contiguous():
            x = x.contiguous()
        return x.data_ptr(), x
    a = np.ascontiguousarray(x, dtype=dtype)
    if shape_tail is not None and a.shape[1:] != shape_tail:
        a = a.reshape((-1,) + shape_tail)
    return a.ctypes.data, a


def _out(out: Any, shape, dtype) -> tuple[int, Any]:
    if out is None:
        out = np.empty(shape, dtype=dtype)
    if _is_torch(out):
        return out.data_ptr(), out
    return out.ctypes.data, out


def _n(x: Any) -> int:
    return int(x.shape[0])


class _CudaFrame:
    """__cuda_array_interface__ view of a library-owned device frame."""

    def __init__(self, ptr: int, height: int, width: int, ctx, owner: bool):
        self.ptr, self.shape, self.ctx, self.owner = ptr, (height, width, 3), ctx, owner
        self.__cuda_array_interface__ = {"shape": self.shape, "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}

    def release(self):
        if self.ptr:
            lib().pf_ipc_frame_release(self.ctx._h, C.c_void_p(self.ptr), int(self.owner))
            self.ptr = 0


def _device_frame(ptr: int, height: int, width: int, ctx, owner: bool):
    import torch
    holder = _CudaFrame(ptr, height, width, ctx, owner)
    t = torch.as_tensor(holder, device="cuda")
    t._pf_holder = holder  # keeps the mapping alive with the tensor
    return t


# ------------------------------------------------------------- context ----


class Context:
    """One CUDA device; scene, field and photon map are device-resident."""

    def __init__(self, device: int = 0, stream: int | None = None):
        h = C.c_void_p()
        check(lib().pf_ctx_create(device, C.byref(h)))
        self._h = h
        self.device = device
        self.field_config: FieldConfig | None = None
        self.n_lights = 0
        if stream is not None:
            self.set_stream(stream)

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().pf_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_stream(self, cuda_stream: int | None) -> None:
        check(lib().pf_ctx_set_stream(self._h, C.c_void_p(cuda_stream or 0)))

    def synchronize(self) -> None:
        check(lib().pf_ctx_synchronize(self._h))

    def set_timing(self, on: bool) -> None:
        check(lib().pf_ctx_set_timing(self._h, int(on)))

    # ---- scene
    def upload_volume(self, v) -> None:
        """VolumeGrid(nx, ny, nz, data): v has shape (nz, ny, nx), x fastest."""
        p, keep = _in(v, np.float32)
        nz, ny, nx = keep.shape
        check(lib().pf_volume_upload(self._h, nx, ny, nz, p))

    def set_medium(self, tf_points, density_scale: float = 100.0,
                   sigma_max: float = -1.0) -> float:
        tf = validate_tf(tf_points)
        check(lib().pf_medium_set(self._h, tf.ctypes.data, tf.shape[0], float(density_scale),
                                  float(sigma_max)))
        return self.sigma_max

    @property
    def sigma_max(self) -> float:
        v = C.c_double()
        check(lib().pf_medium_sigma_max(self._h, C.byref(v)))
        return v.value

    def set_lights(self, lights) -> None:
        a = np.ascontiguousarray(lights, dtype=np.float64).reshape(-1, 6)
        check(lib().pf_lights_set(self._h, a.ctypes.data, a.shape[0]))
        self.n_lights = a.shape[0]

    # ---- field
    def load_field(self, cfg: FieldConfig, params) -> None:
        p, keep = _in(params, np.float32)
        check(lib().pf_field_load(self._h, C.byref(cfg.c()), p, int(np.prod(keep.shape))))
        self.field_config = cfg

    # ---- training
    def train_init(self, cfg: FieldConfig, params, adam: AdamConfig | None = None) -> None:
        p, keep = _in(params, np.float32)
        check(lib().pf_train_init(self._h, C.byref(cfg.c()), p, int(np.prod(keep.shape)),
                                  C.byref(adam.c()) if adam is not None else None))
        self.field_config = cfg
        self.adam_config = adam

    def train_counts(self) -> tuple[int, int]:
        a, b = C.c_size_t(), C.c_size_t()
        check(lib().pf_train_counts(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def _batch(self, x3, wsph2, g, targets3):
        px, kx = _in(x3, np.float32)
        pw, kw = _in(wsph2, np.float32)
        pg, kg = _in(g, np.float32)
        pt, kt = _in(targets3, np.float32)
        return _n(kx), (px, pw, pg, pt), (kx, kw, kg, kt)

    def train_step(self, x3, wsph2, g, targets3, step: int, total_steps: int) -> float:
        n, ptrs, keep = self._batch(x3, wsph2, g, targets3)
        loss = C.c_double()
        check(lib().pf_train_step(self._h, n, *ptrs, int(step), int(total_steps), C.byref(loss)))
        return loss.value

    def train_grad(self, x3, wsph2, g, targets3):
        """Parity entry: (loss, dense binary32 gradient, touched flags per table entry)."""
        n, ptrs, keep = self._batch(x3, wsph2, g, targets3)
        n_params, n_entries = self.train_counts()
        grad = np.zeros(n_params, np.float32)
        touched = np.zeros(n_entries, np.uint8)
        loss = C.c_double()
        check(lib().pf_train_grad(self._h, n, *ptrs, C.byref(loss), grad.ctypes.data, touched.ctypes.data))
        return loss.value, grad, touched

    # ---- data-parallel training: backward -> all-reduce -> apply
    def train_backward(self, x3, wsph2, g, targets3, n_global: int) -> float:
        """This rank's shard of a step; returns its part of the global loss."""
        n, ptrs, keep = self._batch(x3, wsph2, g, targets3)
        loss = C.c_double()
        check(lib().pf_train_backward(self._h, n, *ptrs, int(n_global), C.byref(loss)))
        return loss.value

    def train_grad_tensors(self):
        """Zero-copy CUDA views of the gradient state: (int64 table gradient in
        2^-40 fixed point, float32 MLP gradient, uint8 touched flags)."""
        import torch
        gt, gm, tc = C.c_void_p(), C.c_void_p(), C.c_void_p()
        nt, nm, ne = C.c_size_t(), C.c_size_t(), C.c_size_t()
        check(lib().pf_train_grad_buffers(self._h, C.byref(gt), C.byref(nt), C.byref(gm), C.byref(nm), C.byref(tc),
                                          C.byref(ne)))

        class _V:
            def __init__(self, ptr, n, ts):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": ts, "data": (ptr, False), "version": 3}

        return (torch.as_tensor(_V(gt.value, nt.value, "<i8"), device="cuda"),
                torch.as_tensor(_V(gm.value, nm.value, "<f4"), device="cuda"),
                torch.as_tensor(_V(tc.value, ne.value, "|u1"), device="cuda"))

    def train_apply(self, step: int, total_steps: int) -> None:
        check(lib().pf_train_apply(self._h, int(step), int(total_steps)))

    def train_params(self) -> np.ndarray:
        n_params, _ = self.train_counts()
        out = np.zeros(n_params, np.float32)
        check(lib().pf_train_params(self._h, out.ctypes.data, n_params))
        return out

    def train_commit(self) -> None:
        check(lib().pf_train_commit(self._h))

    def train(self, cfg: TrainConfig, start_step: int = 0, stop_step: int | None = None) -> TrainResult:
        """train(field, map, cfg) on the resident photon map,
        steps [start_step, stop_step or total).  start_step > 0 continues a run
        restored by train_load (its next step): schedule radius, query streams,
        lr and Adam bias correction use the absolute step, so train(stop=k) ->
        train_save -> train_load -> train(start=k) reproduces the uninterrupted
        run bit for bit.  The result covers the steps run."""
        ends = np.ascontiguousarray(cfg.schedule_ends, np.float64)
        radii = np.ascontiguousarray(cfg.schedule_radii, np.float64)
        d = _lib.TrainDesc(int(cfg.total_steps), int(cfg.batch_size), int(cfg.K), len(ends), ends.ctypes.data,
                           radii.ctypes.data, float(cfg.psi), int(cfg.seed), int(start_step),
                           int(stop_step or 0))
        n, s0 = int(cfg.total_steps), int(start_step)
        s1 = int(stop_step) if stop_step else n
        hist, ka, kb = np.zeros(n), np.zeros(n), np.zeros(n)
        a, b = C.c_double(), C.c_double()
        check(lib().pf_train(self._h, C.byref(d), hist.ctypes.data, C.byref(a), C.byref(b), ka.ctypes.data,
                             kb.ctypes.data))
        radius = np.array([schedule_radius(cfg.schedule_ends, cfg.schedule_radii, s, n) for s in range(s0, s1)])
        lrs = np.array([lr_at(s, n, getattr(self, "adam_config", None)) for s in range(s0, s1)])
        return TrainResult(hist[s0:s1], a.value, b.value, ka[s0:s1], kb[s0:s1], radius, lrs, first_step=s0)

    def train_state(self):
        """(params, m, v) of the optimizer, binary32."""
        n_params, _ = self.train_counts()
        out = [np.zeros(n_params, np.float32) for _ in range(3)]
        check(lib().pf_train_state_get(self._h, *[o.ctypes.data for o in out], n_params))
        return tuple(out)

    def train_save(self, path, phase_set, next_step: int, total_steps: int = 0) -> None:
        p, m, v = self.train_state()
        save_checkpoint(path, self.field_config, phase_set, next_step, p, m, v,
                        adam=getattr(self, "adam_config", None), total_steps=total_steps)

    def train_load(self, path, adam: "AdamConfig | None" = None):
        """Restore a checkpoint bit-exactly (binary32 state stored as binary64);
        returns (FieldConfig, phase_set, next step).  The Adam hyperparameters
        come from the checkpoint unless `adam` overrides them."""
        cfg, gs, step, (p, m, v), ck_adam, _ = _parse_checkpoint(path)
        if adam is None:
            adam = ck_adam
        p32, m32, v32 = (np.ascontiguousarray(x, np.float32) for x in (p, m, v))
        if not (np.array_equal(p32.astype(np.float64), p) and np.array_equal(m32.astype(np.float64), m)
                and np.array_equal(v32.astype(np.float64), v)):
            raise ValueError("field checkpoint: state is not binary32-representable")
        self.train_init(cfg, p32, adam)
        check(lib().pf_train_state_set(self._h, p32.ctypes.data, m32.ctypes.data, v32.ctypes.data, len(p32)))
        return cfg, gs, step

    def field_query(self, x3, wsph2, g, decoded: bool = True, out=None):
        px, kx = _in(x3, np.float32)
        pw, kw = _in(wsph2, np.float32)
        pg, kg = _in(g, np.float32)
        n = _n(kx)
        po, out = _out(out, (n, 3), np.float32)
        check(lib().pf_field_query(self._h, n, px, pw, pg, po, int(decoded)))
        return out

    # ---- render
    @staticmethod
    def camera(spec: CameraSpec) -> _lib.Camera:
        cam = _lib.Camera()
        pos = (C.c_double * 3)(*spec.position)
        at = (C.c_double * 3)(*spec.look_at)
        up = (C.c_double * 3)(*spec.up)
        check(lib().pf_camera_make(pos, at, up, float(spec.vfov_deg), spec.width, spec.height,
                                   C.byref(cam)))
        return cam

    def render_neural(self, cam: _lib.Camera | CameraSpec, cfg: RenderConfig, out=None,
                      stats: bool = False):
        if isinstance(cam, CameraSpec):
            cam = self.camera(cam)
        po, out = _out(out, (cam.height, cam.width, 3), np.float32)
        st = _lib.RenderStats()
        check(lib().pf_render_neural(self._h, C.byref(cam), C.byref(cfg.c()), po,
                                     C.byref(st) if stats else None))
        if stats:
            return out, {k: getattr(st, k) for k, _ in _lib.RenderStats._fields_}
        return out

    def render_neural_async(self, cam: _lib.Camera | CameraSpec, cfg: RenderConfig, out):
        """Enqueue a frame into HOST memory `out` (pinned for overlap) and return;
        `out` is complete after frame_wait(out) / synchronize()."""
        if isinstance(cam, CameraSpec):
            cam = self.camera(cam)
        po, out = _out(out, (cam.height, cam.width, 3), np.float32)
        check(lib().pf_render_neural_async(self._h, C.byref(cam), C.byref(cfg.c()), po))
        return out

    def frame_wait(self, out) -> None:
        po, _ = _out(out, None, np.float32)
        check(lib().pf_frame_wait(self._h, po))

    def render_path_traced(self, cam: _lib.Camera | CameraSpec, cfg: RenderConfig,
                           path: PathTraceConfig | None = None, out=None, stats: bool = False):
        """render_path_traced: NEE at every vertex, HG continuation."""
        if isinstance(cam, CameraSpec):
            cam = self.camera(cam)
        path = path or PathTraceConfig()
        po, out = _out(out, (cam.height, cam.width, 3), np.float32)
        st = _lib.RenderStats()
        check(lib().pf_render_path_traced(self._h, C.byref(cam), C.byref(cfg.c()), C.byref(path.c()), po,
                                          C.byref(st) if stats else None))
        if stats:
            return out, {k: getattr(st, k) for k, _ in _lib.RenderStats._fields_}
        return out

    def render_photon_map(self, cam: _lib.Camera | CameraSpec, cfg: RenderConfig, K: int = 64,
                          r_max: float = float("inf"), out=None, stats: bool = False):
        """render_photon_map: L_i from Eq. 6 over the resident map."""
        if isinstance(cam, CameraSpec):
            cam = self.camera(cam)
        po, out = _out(out, (cam.height, cam.width, 3), np.float32)
        st = _lib.RenderStats()
        check(lib().pf_render_photon_map(self._h, C.byref(cam), C.byref(cfg.c()), int(K), float(r_max), po,
                                         C.byref(st) if stats else None))
        if stats:
            return out, {k: getattr(st, k) for k, _ in _lib.RenderStats._fields_}
        return out

    # ---- multi-GPU frame over NVLink peer memory (CUDA IPC)
    def ipc_frame_create(self, height: int, width: int):
        """rank 0: a device frame other ranks can map; returns (tensor, 64-byte handle)."""
        ptr, h = C.c_void_p(), (C.c_uint8 * 64)()
        check(lib().pf_ipc_frame_create(self._h, height * width * 12, C.byref(ptr), h))
        return _device_frame(ptr.value, height, width, self, owner=True), bytes(h)

    def ipc_frame_open(self, handle: bytes, height: int, width: int):
        """rank > 0: map rank 0's frame; renders with out= this tensor store into it."""
        ptr, h = C.c_void_p(), (C.c_uint8 * 64).from_buffer_copy(handle)
        check(lib().pf_ipc_frame_open(self._h, h, C.byref(ptr)))
        return _device_frame(ptr.value, height, width, self, owner=False)

    def tiles_count(self, cam: _lib.Camera, cfg: RenderConfig, shard: int) -> int:
        n = C.c_int()
        check(lib().pf_tiles_count(C.byref(cam), C.byref(cfg.c()), shard, C.byref(n)))
        return n.value

    def tiles_pack(self, cam, cfg: RenderConfig, frame, packed) -> None:
        check(lib().pf_tiles_pack(self._h, C.byref(cam), C.byref(cfg.c()), frame.data_ptr(),
                                  packed.data_ptr()))

    def tiles_unpack(self, cam, cfg: RenderConfig, packed_all, per_shard: int, frame) -> None:
        check(lib().pf_tiles_unpack(self._h, C.byref(cam), C.byref(cfg.c()),
                                    packed_all.data_ptr(), per_shard, frame.data_ptr()))

    # ---- parity entry points
    def delta_track_batch(self, o3, d3, tmin, tmax, seed: int, stream: str | int, idx,
                          fp64: bool = True, with_scalar: bool = False):
        """pf::delta_track per ray (volume.cpp:204-225) -> (hit, position, albedo), or
        (hit, position, scalar, albedo) = Interaction{position, scalar, albedo}
        with with_scalar=True."""
        po, ko = _in(o3, np.float64)
        pd, kd = _in(d3, np.float64)
        p0, k0 = _in(tmin, np.float64)
        p1, k1 = _in(tmax, np.float64)
        pi, ki = _in(idx, np.uint64)
        n = _n(ko)
        ph, hit = _out(None, (n,), np.int32)
        pp, pos = _out(None, (n, 3), np.float64)
        pr, rgba = _out(None, (n, 4), np.float64)
        psc, scalar = _out(None, (n,), np.float64)
        s = STREAM[stream] if isinstance(stream, str) else int(stream)
        check(lib().pf_delta_track_batch(self._h, n, po, pd, p0, p1, seed, s, pi, int(fp64), ph,
                                         pp, psc, pr))
        return (hit, pos, scalar, rgba) if with_scalar else (hit, pos, rgba)

    def transmittance_batch(self, a3, b3, seed: int, stream: str | int, idx, n_trials: int = 1,
                            ratio: bool = False):
        pa, ka = _in(a3, np.float64)
        pb, kb = _in(b3, np.float64)
        pi, ki = _in(idx, np.uint64)
        n = _n(ka)
        po, out = _out(None, (n,), np.float64)
        s = STREAM[stream] if isinstance(stream, str) else int(stream)
        fn = lib().pf_transmittance_ratio_batch if ratio else lib().pf_transmittance_batch
        check(fn(self._h, n, pa, pb, seed, s, pi, n_trials, po))
        return out

    def rng_doubles(self, seed: int, stream: str | int, idx, n_draws: int):
        pi, ki = _in(idx, np.uint64)
        n = _n(ki)
        po, out = _out(None, (n, n_draws), np.float64)
        s = STREAM[stream] if isinstance(stream, str) else int(stream)
        check(lib().pf_rng_doubles(self._h, n, seed, s, pi, n_draws, po))
        return out

    # ---- photon tracing (Alg. 1)
    def trace_photons(self, tc: TraceConfig, device: bool = False) -> TraceResult:
        """trace_photons on the device; photons come back to the host unless
        device=True (then a uint8 CUDA tensor [n, 40] in the pf_photon layout)."""
        gs = np.ascontiguousarray(tc.phase_set, dtype=np.float64)
        d = _lib.TraceDesc(int(tc.n_total), len(gs), gs.ctypes.data, int(tc.max_bounces),
                           int(tc.rr_start_bounce), float(tc.rr_min_survival),
                           float(tc.rr_max_survival), int(tc.seed))
        n_l = self.n_lights
        emitted = np.zeros(max(1, n_l * len(gs)), np.uint64)
        n = C.c_size_t(0)
        check(lib().pf_trace_photons(self._h, C.byref(d), C.byref(n), emitted.ctypes.data))
        n = n.value
        if device:
            import torch
            out = torch.empty((n, 40), dtype=torch.uint8, device=f"cuda:{self.device}")
            check(lib().pf_trace_fetch(self._h, out.data_ptr() if n else None, n))
        else:
            out = np.zeros(n, dtype=PHOTON_DTYPE)
            check(lib().pf_trace_fetch(self._h, out.ctypes.data if n else None, n))
        return TraceResult(out, list(gs), emitted[: n_l * len(gs)], n_l)

    def trace_path_counts(self, n_total: int) -> np.ndarray:
        out = np.zeros(max(1, n_total), np.uint32)
        check(lib().pf_trace_path_counts(self._h, out.ctypes.data, n_total))
        return out[:n_total]

    def trace_stats(self) -> dict:
        a, b, st = C.c_double(), C.c_double(), C.c_uint64()
        check(lib().pf_trace_stats(self._h, C.byref(a), C.byref(b), C.byref(st)))
        return {"ms_trace": a.value, "ms_compact": b.value, "tentative_collisions": st.value}

    def knn_build_traced(self, phase_set) -> None:
        """KNN build straight from the resident trace (no host round trip)."""
        ps = np.ascontiguousarray(phase_set, dtype=np.float64)
        check(lib().pf_knn_build_traced(self._h, len(ps), ps.ctypes.data))
        self.phase_set = ps

    # ---- photon map / KNN
    def knn_build(self, photons, phase_set) -> None:
        if _is_torch(photons):
            n = photons.numel() // 40
            p, keep = photons.data_ptr(), photons
        else:
            a = np.ascontiguousarray(photons, dtype=PHOTON_DTYPE)
            n, p, keep = len(a), a.ctypes.data, a
        ps = np.ascontiguousarray(phase_set, dtype=np.float64)
        check(lib().pf_knn_build(self._h, p, n, len(ps), ps.ctypes.data))
        self.phase_set = ps

    def knn_query(self, x3, gidx, K: int, r_max: float = float("inf")):
        px, kx = _in(x3, np.float32)
        pg, kg = _in(gidx, np.uint8)
        n = _n(kx)
        pi, ids = _out(None, (n, K), np.uint32)
        pd, d2 = _out(None, (n, K), np.float32)
        pc, cnt = _out(None, (n,), np.int32)
        check(lib().pf_knn_query(self._h, n, px, pg, K, float(r_max), pi, pd, pc))
        return ids, d2, cnt

    def knn_targets(self, x3, w3, gidx, K: int, r_max: float = float("inf"), psi: float = 5.0,
                    with_ids: bool = False):
        px, kx = _in(x3, np.float32)
        pw, kw = _in(w3, np.float64)
        pg, kg = _in(gidx, np.uint8)
        n = _n(kx)
        pt, tg = _out(None, (n, 3), np.float64)
        if with_ids:
            pi, ids = _out(None, (n, K), np.uint32)
            pd, d2 = _out(None, (n, K), np.float32)
            pc, cnt = _out(None, (n,), np.int32)
        else:
            pi = pd = pc = None
        check(lib().pf_knn_targets(self._h, n, px, pw, pg, K, float(r_max), float(psi), pt, pi,
                                   pd, pc))
        return (tg, ids, d2, cnt) if with_ids else tg

    def make_batch(self, seed: int, step: int, batch: int, K: int,
                   r_max: float = float("inf"), psi: float = 5.0):
        px, x = _out(None, (batch, 3), np.float32)
        pw, w = _out(None, (batch, 3), np.float64)
        pg, g = _out(None, (batch,), np.uint8)
        pt, t = _out(None, (batch, 3), np.float64)
        check(lib().pf_make_batch(self._h, seed, step, batch, K, float(r_max), float(psi), px,
                                  pw, pg, pt))
        return x, w, g, t


def schedule_radius(ends, radii, step: int, total: int) -> float:
    """KnnSchedule lookup: first segment whose end >= (step+1)/total."""
    progress = (step + 1) / total
    for e, r in zip(ends, radii):
        if e >= progress:
            return float(r)
    return float(radii[-1])
