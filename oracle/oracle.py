"""ctypes wrapper of the CPU ORACLE (TEST INFRASTRUCTURE ONLY).

Loaded only by tests/, __graft_entry__.smoke() (as the checker) and bench.py's
cpu_baseline / --impl reference leg.  Two libraries:
  oracle/liboracle.so     -- the C restatement (pf_oracle.c), always buildable
  oracle/_ref/libpfref.so -- the UNMODIFIED reference sources + ref_shim.cpp;
                             built here only when /root/reference exists, then
                             shipped prebuilt (it is git-ignored, not gpurun-ignored)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libpfref.so"
REF_SRC = Path(os.environ.get("PF_REFERENCE", "/root/reference"))


def build(ref: bool | None = None) -> None:
    """make -C oracle (the C restatement; + _ref when the reference is present)."""
    targets = [str(LIB)]
    if ref is None:
        ref = (REF_SRC / "proj" / "src" / "volume.cpp").exists()
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE), f"REF={REF_SRC}", *targets], check=True,
                   capture_output=True)


class Grid(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("data", C.c_void_p),
                ("value_min", C.c_float), ("value_max", C.c_float)]


class Tf(C.Structure):
    _fields_ = [("n", C.c_int), ("pts", C.c_void_p)]


class Medium(C.Structure):
    _fields_ = [("grid", Grid), ("tf", Tf), ("density_scale", C.c_double),
                ("sigma_max", C.c_double)]


class HashCfg(C.Structure):
    _fields_ = [("dims", C.c_int), ("levels", C.c_int), ("features", C.c_int),
                ("base_res", C.c_int), ("growth", C.c_double), ("log2_table", C.c_int)]


class FieldCfg(C.Structure):
    _fields_ = [("pos", HashCfg), ("dir", HashCfg), ("hidden_layers", C.c_int), ("width", C.c_int),
                ("psi", C.c_double)]


class Camera(C.Structure):
    _fields_ = [("origin", C.c_double * 3), ("forward", C.c_double * 3), ("right", C.c_double * 3),
                ("up", C.c_double * 3), ("width", C.c_int), ("height", C.c_int)]


class Light(C.Structure):
    _fields_ = [("pos", C.c_double * 3), ("intensity", C.c_double * 3)]


class RenderCfg(C.Structure):
    _fields_ = [("spp", C.c_int), ("g", C.c_double), ("seed", C.c_uint64), ("w_d", C.c_double),
                ("w_i", C.c_double), ("background", C.c_double * 3), ("nee_trials", C.c_int),
                ("use_field", C.c_int), ("x0", C.c_int), ("y0", C.c_int), ("x1", C.c_int),
                ("y1", C.c_int)]


class TraceCfg(C.Structure):
    _fields_ = [("n_total", C.c_uint64), ("n_phases", C.c_int), ("phase_set", C.c_void_p),
                ("max_bounces", C.c_int), ("rr_start_bounce", C.c_int), ("rr_min_survival", C.c_double),
                ("rr_max_survival", C.c_double), ("seed", C.c_uint64)]


class RenderStats(C.Structure):
    _fields_ = [("samples", C.c_uint64), ("hits", C.c_uint64)]


class AdamCfg(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("decay", C.c_double), ("decay_start", C.c_double), ("decay_interval", C.c_int)]


class PtCfg(C.Structure):
    _fields_ = [("max_bounces", C.c_int), ("rr_start_bounce", C.c_int), ("rr_min_survival", C.c_double),
                ("rr_max_survival", C.c_double)]


class PmSrc(C.Structure):
    _fields_ = [("ph", C.c_void_p), ("n", C.c_size_t), ("tree", C.c_void_p), ("g_index", C.c_int),
                ("K", C.c_int), ("r_max", C.c_float)]


_P = C.c_void_p
_SIG = {
    "or_next_u32": (C.c_uint32, [_P]),
    "or_next_double": (C.c_double, [_P]),
    "or_make_rng": (None, [_P, C.c_uint64, C.c_uint64, C.c_uint64]),
    "or_splitmix64": (C.c_uint64, [C.c_uint64]),
    "or_hg_eval": (C.c_double, [C.c_double, C.c_double]),
    "or_aabb_intersect": (C.c_int, [_P, _P, C.c_double, C.c_double, _P, _P]),
    "or_grid_init": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, _P]),
    "or_grid_sample": (C.c_double, [_P, _P]),
    "or_tf_classify": (None, [_P, C.c_double, _P]),
    "or_medium_init": (C.c_int, [_P, _P, _P, C.c_double]),
    "or_delta_track_batch": (C.c_int, [_P, C.c_size_t, _P, _P, _P, _P, C.c_uint64, C.c_uint64, _P,
                                       _P, _P, _P, _P]),
    "or_transmittance_batch": (None, [_P, C.c_size_t, _P, _P, C.c_uint64, C.c_uint64, _P, C.c_int,
                                      _P]),
    "or_rng_doubles": (None, [C.c_uint64, C.c_uint64, C.c_size_t, _P, C.c_int, _P]),
    "or_field_param_count": (C.c_size_t, [_P]),
    "or_field_init": (None, [_P, C.c_uint64, C.c_double, C.c_double, _P]),
    "or_hashgrid_param_count": (C.c_size_t, [_P]),
    "or_field_input_dim": (C.c_int, [_P]),
    "or_field_encode": (None, [_P, _P, _P, _P, C.c_double, _P]),
    "or_field_forward": (None, [_P, _P, C.c_size_t, _P, _P, _P, _P]),
    "or_field_infer": (None, [_P, _P, C.c_size_t, _P, _P, _P, _P]),
    "or_dir_to_sph": (None, [_P, _P]),
    "or_encode_log": (C.c_double, [C.c_double, C.c_double]),
    "or_decode_log": (C.c_double, [C.c_double, C.c_double]),
    "or_knn_brute": (C.c_int, [_P, C.c_size_t, _P, C.c_int, C.c_int, C.c_float, _P, _P]),
    "or_kd_build": (C.c_void_p, [_P, C.c_size_t]),
    "or_kd_free": (None, [_P]),
    "or_kd_knn": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_float, _P, _P]),
    "or_estimate_radiance": (None, [_P, _P, _P, C.c_int, _P, C.c_double, _P]),
    "or_make_queries": (None, [C.c_uint64, C.c_uint64, C.c_size_t, C.c_int, _P, _P, _P]),
    "or_schedule_radius": (C.c_double, [_P, _P, C.c_int, C.c_uint64, C.c_uint64]),
    "or_knn_targets": (None, [_P, _P, C.c_size_t, _P, _P, _P, _P, C.c_int, C.c_float, C.c_double,
                              _P, _P, _P, _P]),
    "or_camera_make": (None, [_P, _P, _P, _P, C.c_double, C.c_int, C.c_int]),
    "or_render_neural": (None, [_P, _P, C.c_int, _P, _P, _P, _P, _P, _P]),
    "or_lr_at": (C.c_double, [_P, C.c_uint64, C.c_uint64]),
    "or_train_grad": (C.c_double, [_P, _P, C.c_size_t, _P, _P, _P, _P, C.c_double, _P, _P, _P, _P]),
    "or_adam_update": (None, [_P, _P, _P, _P, _P, _P, _P, C.c_uint64, C.c_uint64]),
    "or_render_path_traced": (None, [_P, _P, C.c_int, _P, _P, _P, _P, _P]),
    "or_render_photon_map": (None, [_P, _P, C.c_int, _P, _P, _P, _P, _P]),
    "or_hg_sample_cos": (C.c_double, [C.c_double, C.c_double]),
    "or_hg_sample": (None, [C.c_double, _P, C.c_double, C.c_double, _P]),
    "or_from_local_frame": (None, [_P, _P, _P]),
    "or_emit_direction": (None, [_P, _P, _P]),
    "or_trace_photons": (C.c_size_t, [_P, _P, C.c_int, _P, _P, C.c_size_t, _P, _P]),
}

_REF_SIG = {
    "ref_last_error": (C.c_char_p, []),
    "ref_trace_photons": (C.c_size_t, [_P, _P, C.c_int, C.c_uint64, C.c_int, _P, C.c_int, C.c_int,
                                       C.c_double, C.c_double, C.c_uint64, _P, _P, C.c_size_t]),
    "ref_rng_u32": (None, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, _P]),
    "ref_rng_double": (None, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, _P]),
    "ref_splitmix64": (C.c_uint64, [C.c_uint64]),
    "ref_hg_eval": (C.c_double, [C.c_double, C.c_double]),
    "ref_hg_sample_cos": (C.c_double, [C.c_double, C.c_double]),
    "ref_hg_cdf": (C.c_double, [C.c_double, C.c_double]),
    "ref_hg_sample": (None, [C.c_double, _P, C.c_double, C.c_double, _P]),
    "ref_aabb_intersect": (C.c_int, [_P, _P, C.c_double, C.c_double, _P, _P]),
    "ref_scene_create": (C.c_int, [C.c_int, C.c_int, C.c_int, _P, _P, C.c_int, C.c_double,
                                   C.POINTER(C.c_void_p)]),
    "ref_scene_destroy": (None, [_P]),
    "ref_scene_sigma_max": (C.c_double, [_P]),
    "ref_grid_sample": (C.c_double, [_P, _P]),
    "ref_tf_classify": (None, [_P, C.c_double, _P]),
    "ref_delta_track_batch": (C.c_int, [_P, C.c_size_t, _P, _P, _P, _P, C.c_uint64, C.c_uint64,
                                        _P, _P, _P, _P, _P]),
    "ref_transmittance_batch": (C.c_int, [_P, C.c_size_t, _P, _P, C.c_uint64, C.c_uint64, _P,
                                          C.c_int, _P]),
    "ref_render_neural": (C.c_int, [_P, _P, C.c_int, _P, _P, _P, _P, C.c_int, _P, _P]),
    "ref_render_path_traced": (C.c_int, [_P, _P, C.c_int, _P, _P, _P, C.c_int, _P, _P]),
}

_lib = None
_ref = None


def _stale(out: Path, *srcs: Path) -> bool:
    if not out.exists():
        return True
    have = [p for p in srcs if p.exists()]
    return bool(have) and out.stat().st_mtime < max(p.stat().st_mtime for p in have)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if _stale(LIB, HERE / "pf_oracle.c", HERE / "pf_oracle.h"):
            build(ref=False)
        L = C.CDLL(str(LIB))
        for k, (r, a) in _SIG.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _lib = L
    return _lib


def ref_available() -> bool:
    return REF_LIB.exists() or (REF_SRC / "proj" / "src" / "volume.cpp").exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_LIB.exists() or ((REF_SRC / "proj").exists() and _stale(
                REF_LIB, HERE / "ref_shim.cpp", HERE / "pf_oracle.c", HERE / "pf_oracle.h")):
            build(ref=True)
        L = C.CDLL(str(REF_LIB))
        for k, (r, a) in _REF_SIG.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _ref = L
    return _ref


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


# ------------------------------------------------------------ scene ------


class OracleScene:
    """A medium (grid + TF + density) for the C restatement."""

    def __init__(self, vol: np.ndarray, tf: np.ndarray, density_scale: float = 100.0):
        self.vol = np.ascontiguousarray(vol, dtype=np.float32)
        self.tf = np.ascontiguousarray(tf, dtype=np.float64)
        nz, ny, nx = self.vol.shape
        self.grid = Grid()
        if lib().or_grid_init(C.byref(self.grid), nx, ny, nz, _p(self.vol)):
            raise ValueError("VolumeGrid: invalid")
        self.tfs = Tf(self.tf.shape[0], _p(self.tf))
        self.medium = Medium()
        if lib().or_medium_init(C.byref(self.medium), C.byref(self.grid), C.byref(self.tfs),
                                density_scale):
            raise ValueError("Medium: invalid density scale")

    @property
    def sigma_max(self) -> float:
        return self.medium.sigma_max

    def delta_track(self, o, d, tmin, tmax, seed, stream, idx, with_scalar=False):
        o = np.ascontiguousarray(o, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        tmin = np.ascontiguousarray(tmin, np.float64)
        tmax = np.ascontiguousarray(tmax, np.float64)
        idx = np.ascontiguousarray(idx, np.uint64)
        n = len(idx)
        hit = np.zeros(n, np.int32)
        pos = np.zeros((n, 3))
        sc = np.zeros(n)
        rgba = np.zeros((n, 4))
        if lib().or_delta_track_batch(C.byref(self.medium), n, _p(o), _p(d), _p(tmin), _p(tmax),
                                      seed, stream, _p(idx), _p(hit), _p(pos), _p(sc), _p(rgba)):
            raise ValueError("delta_track: invalid ray")
        return (hit, pos, sc, rgba) if with_scalar else (hit, pos, rgba)

    def transmittance(self, a, b, seed, stream, idx, n_trials=1):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        idx = np.ascontiguousarray(idx, np.uint64)
        out = np.zeros(len(idx))
        lib().or_transmittance_batch(C.byref(self.medium), len(idx), _p(a), _p(b), seed, stream,
                                     _p(idx), n_trials, _p(out))
        return out

    def sample(self, p) -> float:
        p = np.ascontiguousarray(p, np.float64)
        return lib().or_grid_sample(C.byref(self.grid), _p(p))


class RefScene:
    """The same medium through the UNMODIFIED reference (oracle/_ref)."""

    def __init__(self, vol: np.ndarray, tf: np.ndarray, density_scale: float = 100.0):
        self.vol = np.ascontiguousarray(vol, dtype=np.float32)
        self.tf = np.ascontiguousarray(tf, dtype=np.float64)
        nz, ny, nx = self.vol.shape
        h = C.c_void_p()
        if ref().ref_scene_create(nx, ny, nz, _p(self.vol), _p(self.tf), self.tf.shape[0],
                                  density_scale, C.byref(h)):
            raise ValueError(ref().ref_last_error().decode())
        self.h = h

    def __del__(self):
        try:
            ref().ref_scene_destroy(self.h)
        except Exception:
            pass

    @property
    def sigma_max(self) -> float:
        return ref().ref_scene_sigma_max(self.h)

    def delta_track(self, o, d, tmin, tmax, seed, stream, idx, with_scalar=False):
        o = np.ascontiguousarray(o, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        tmin = np.ascontiguousarray(tmin, np.float64)
        tmax = np.ascontiguousarray(tmax, np.float64)
        idx = np.ascontiguousarray(idx, np.uint64)
        n = len(idx)
        hit = np.zeros(n, np.int32)
        pos = np.zeros((n, 3))
        sc = np.zeros(n)
        rgba = np.zeros((n, 4))
        if ref().ref_delta_track_batch(self.h, n, _p(o), _p(d), _p(tmin), _p(tmax), seed, stream,
                                       _p(idx), _p(hit), _p(pos), _p(sc), _p(rgba)):
            raise ValueError(ref().ref_last_error().decode())
        return (hit, pos, sc, rgba) if with_scalar else (hit, pos, rgba)

    def transmittance(self, a, b, seed, stream, idx, n_trials=1):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        idx = np.ascontiguousarray(idx, np.uint64)
        out = np.zeros(len(idx))
        if ref().ref_transmittance_batch(self.h, len(idx), _p(a), _p(b), seed, stream, _p(idx),
                                         n_trials, _p(out)):
            raise ValueError(ref().ref_last_error().decode())
        return out


# ------------------------------------------------------------ field ------


def field_cfg(fc) -> FieldCfg:
    """From paper_2304_07338_b200.FieldConfig (duck-typed)."""
    def h(g):
        return HashCfg(g.dims, g.levels, g.features, g.base_res, float(g.growth), g.log2_table)
    return FieldCfg(h(fc.pos), h(fc.dir), fc.hidden_layers, fc.width, float(fc.psi))


def field_param_count(fc) -> int:
    return lib().or_field_param_count(C.byref(field_cfg(fc)))


def field_init(fc, seed=0, embed_scale=1e-4, bias_scale=0.0) -> np.ndarray:
    """Deterministic parameters in pf_field_init's draw order,
    computed on the CPU so the reference arm never loads the GPU library."""
    out = np.empty(field_param_count(fc), np.float32)
    lib().or_field_init(C.byref(field_cfg(fc)), seed, float(embed_scale), float(bias_scale), _p(out))
    return out


def field_forward(fc, params, x3, w2, g, decoded=False) -> np.ndarray:
    cfg = field_cfg(fc)
    params = np.ascontiguousarray(params, np.float32)
    x3 = np.ascontiguousarray(x3, np.float64)
    w2 = np.ascontiguousarray(w2, np.float64)
    g = np.ascontiguousarray(g, np.float64)
    out = np.zeros((len(g), 3))
    fn = lib().or_field_infer if decoded else lib().or_field_forward
    fn(C.byref(cfg), _p(params), len(g), _p(x3), _p(w2), _p(g), _p(out))
    return out


def field_encode(fc, params, x, w, g) -> np.ndarray:
    cfg = field_cfg(fc)
    params = np.ascontiguousarray(params, np.float32)
    x = np.ascontiguousarray(x, np.float64)
    w = np.ascontiguousarray(w, np.float64)
    out = np.zeros(lib().or_field_input_dim(C.byref(cfg)))
    lib().or_field_encode(C.byref(cfg), _p(params), _p(x), _p(w), float(g), _p(out))
    return out


# -------------------------------------------------------------- KNN ------


class KdTree:
    def __init__(self, photons: np.ndarray):
        self.ph = np.ascontiguousarray(photons)
        assert self.ph.dtype.itemsize == 40
        self.t = lib().or_kd_build(_p(self.ph), len(self.ph))

    def __del__(self):
        try:
            lib().or_kd_free(self.t)
        except Exception:
            pass

    def knn(self, q, g_index, K, r_max=float("inf")):
        q = np.ascontiguousarray(q, np.float32)
        ids = np.zeros(K, np.uint32)
        d2 = np.zeros(K, np.float32)
        n = lib().or_kd_knn(self.t, _p(q), g_index, K, r_max, _p(ids), _p(d2))
        return ids[:n], d2[:n]

    def targets(self, x3, w3, gidx, phase_set, K, r_max, psi):
        x3 = np.ascontiguousarray(x3, np.float32)
        w3 = np.ascontiguousarray(w3, np.float64)
        gidx = np.ascontiguousarray(gidx, np.uint8)
        ps = np.ascontiguousarray(phase_set, np.float64)
        n = len(gidx)
        ids = np.zeros((n, K), np.uint32)
        d2 = np.zeros((n, K), np.float32)
        cnt = np.zeros(n, np.int32)
        tg = np.zeros((n, 3))
        lib().or_knn_targets(self.t, _p(self.ph), n, _p(x3), _p(w3), _p(gidx), _p(ps), K, r_max,
                             psi, _p(ids), _p(d2), _p(cnt), _p(tg))
        return tg, ids, d2, cnt


def knn_brute(photons, q, g_index, K, r_max=float("inf")):
    ph = np.ascontiguousarray(photons)
    q = np.ascontiguousarray(q, np.float32)
    ids = np.zeros(K, np.uint32)
    d2 = np.zeros(K, np.float32)
    n = lib().or_knn_brute(_p(ph), len(ph), _p(q), g_index, K, r_max, _p(ids), _p(d2))
    return ids[:n], d2[:n]


def make_queries(seed, step, batch, n_phases):
    x = np.zeros((batch, 3), np.float32)
    w = np.zeros((batch, 3))
    g = np.zeros(batch, np.uint8)
    lib().or_make_queries(seed, step, batch, n_phases, _p(x), _p(w), _p(g))
    return x, w, g


# ----------------------------------------------------------- render ------


def camera(spec) -> Camera:
    cam = Camera()
    pos = np.array(spec.position, np.float64)
    at = np.array(spec.look_at, np.float64)
    up = np.array(spec.up, np.float64)
    lib().or_camera_make(C.byref(cam), _p(pos), _p(at), _p(up), float(spec.vfov_deg), spec.width,
                         spec.height)
    return cam


def _lights(lights: np.ndarray):
    arr = (Light * len(lights))()
    for i, l in enumerate(lights):
        arr[i].pos[:] = list(l[:3])
        arr[i].intensity[:] = list(l[3:6])
    return arr


def _rcfg(rc, cam, rect):
    x0, y0, x1, y1 = rect if rect is not None else (0, 0, cam.width, cam.height)
    return RenderCfg(rc.spp, float(rc.g), rc.seed, float(rc.w_d), float(rc.w_i),
                     (C.c_double * 3)(*rc.background), rc.nee_trials, int(rc.use_field), x0, y0,
                     x1, y1)


def render_neural(scene: OracleScene, lights, fc, params, cam_spec, rc, rect=None):
    """The C restatement of render_neural (binary64; returns (H, W, 3) float32)."""
    cam = camera(cam_spec)
    ls = _lights(np.asarray(lights, np.float64).reshape(-1, 6))
    cfg = field_cfg(fc) if fc is not None else FieldCfg()
    params = np.ascontiguousarray(params if params is not None else np.zeros(1), np.float32)
    out = np.zeros((cam.height, cam.width, 3), np.float32)
    st = RenderStats()
    lib().or_render_neural(C.byref(scene.medium), ls, len(ls), C.byref(cfg), _p(params),
                           C.byref(cam), C.byref(_rcfg(rc, cam, rect)), _p(out), C.byref(st))
    return out, {"samples": st.samples, "hits": st.hits}


def ref_render_neural(scene: RefScene, lights, fc, params, cam_spec, rc, rect=None, workers=0):
    """The reference CPU path (pf::delta_track/transmittance + parallel_chunks)."""
    cam = camera(cam_spec)
    ls = _lights(np.asarray(lights, np.float64).reshape(-1, 6))
    cfg = field_cfg(fc) if fc is not None else FieldCfg()
    params = np.ascontiguousarray(params if params is not None else np.zeros(1), np.float32)
    out = np.zeros((cam.height, cam.width, 3), np.float32)
    hits = C.c_uint64()
    if ref().ref_render_neural(scene.h, ls, len(ls), C.byref(cfg), _p(params), C.byref(cam),
                               C.byref(_rcfg(rc, cam, rect)), workers or (os.cpu_count() or 1),
                               _p(out), C.byref(hits)):
        raise ValueError(ref().ref_last_error().decode())
    return out, {"hits": hits.value}


# ------------------------------------------------------------ training --


def adam_cfg(a=None) -> AdamCfg:
    """AdamState hyper-parameters; `a` may carry overrides."""
    d = dict(lr=9e-4, beta1=0.9, beta2=0.99, eps=1e-8, decay=0.92, decay_start=0.7, decay_interval=25)
    if a is not None:
        d.update({k: getattr(a, k) for k in d if hasattr(a, k)})
    return AdamCfg(d["lr"], d["beta1"], d["beta2"], d["eps"], d["decay"], d["decay_start"], int(d["decay_interval"]))


def lr_at(step, total, a=None) -> float:
    return lib().or_lr_at(C.byref(adam_cfg(a)), int(step), int(total))


def _mlp_count(fc) -> int:
    din = fc.pos.levels * fc.pos.features + fc.dir.levels * fc.dir.features + 1
    w = fc.width
    return din * w + w + (fc.hidden_layers - 1) * (w * w + w) + 3 * w + 3


def train_grad(fc, params, x3, w2, g, targets3, eps_rel=0.01, want_grad=True, den=None, want_pred=False):
    """rMSE loss and its dense binary64 gradient (or_train_grad); params binary64.
    den (n, 3) freezes the detached denominators; want_pred adds the predictions."""
    cfg = field_cfg(fc)
    params = np.ascontiguousarray(params, np.float64)
    x3 = np.ascontiguousarray(x3, np.float64)
    w2 = np.ascontiguousarray(w2, np.float64)
    g = np.ascontiguousarray(g, np.float64)
    t = np.ascontiguousarray(targets3, np.float64)
    n_ent = _entries(fc)
    grad = np.zeros(len(params)) if want_grad else None
    touched = np.zeros(n_ent, np.uint8) if want_grad else None
    pred = np.zeros((len(g), 3)) if want_pred else None
    den = np.ascontiguousarray(den, np.float64) if den is not None else None
    loss = lib().or_train_grad(C.byref(cfg), _p(params), len(g), _p(x3), _p(w2), _p(g), _p(t), float(eps_rel),
                               _p(grad) if want_grad else None, _p(touched) if want_grad else None,
                               _p(pred) if want_pred else None, _p(den) if den is not None else None)
    if want_pred:
        return loss, grad, touched, pred
    return loss, grad, touched


def _entries(fc) -> int:
    """Table entries (pos then dir), i.e. table parameters / features."""
    n = 0
    for hg in (fc.pos, fc.dir):
        c = HashCfg(hg.dims, hg.levels, hg.features, hg.base_res, float(hg.growth), hg.log2_table)
        n += lib().or_hashgrid_param_count(C.byref(c)) // hg.features
    return n


def adam_update(fc, params, grad, touched, m, v, step, total, a=None):
    """In-place Adam step (or_adam_update) on binary64 params / moments."""
    cfg = field_cfg(fc)
    lib().or_adam_update(C.byref(cfg), C.byref(adam_cfg(a)), _p(params), _p(grad), _p(touched), _p(m), _p(v),
                         int(step), int(total))


def _ptcfg(pt) -> PtCfg:
    return PtCfg(int(pt.max_bounces), int(pt.rr_start_bounce), float(pt.rr_min_survival),
                 float(pt.rr_max_survival))


def render_path_traced(scene: OracleScene, lights, cam_spec, rc, pt, rect=None):
    """render_path_traced on the C restatement: render_neural's
    first interaction + NEE, L_i from a phase-sampled continuation (PathTrace stream)."""
    cam = camera(cam_spec)
    ls = _lights(np.asarray(lights, np.float64).reshape(-1, 6))
    out = np.zeros((cam.height, cam.width, 3), np.float32)
    st = RenderStats()
    lib().or_render_path_traced(C.byref(scene.medium), ls, len(ls), C.byref(cam), C.byref(_rcfg(rc, cam, rect)),
                                C.byref(_ptcfg(pt)), _p(out), C.byref(st))
    return out, {"samples": st.samples, "hits": st.hits}


def ref_render_path_traced(scene: "RefScene", lights, cam_spec, rc, pt, rect=None, workers=0):
    """The same algorithm composed from the reference's own primitives (ref_shim.cpp)."""
    cam = camera(cam_spec)
    ls = _lights(np.asarray(lights, np.float64).reshape(-1, 6))
    out = np.zeros((cam.height, cam.width, 3), np.float32)
    hits = C.c_uint64()
    if ref().ref_render_path_traced(scene.h, ls, len(ls), C.byref(cam), C.byref(_rcfg(rc, cam, rect)),
                                    C.byref(_ptcfg(pt)), workers or (os.cpu_count() or 1), _p(out),
                                    C.byref(hits)):
        raise ValueError(ref().ref_last_error().decode())
    return out, {"hits": hits.value}


def render_photon_map(scene: OracleScene, lights, photons, g_index, K, r_max, cam_spec, rc, rect=None,
                      tree: "KdTree | None" = None):
    """render_photon_map on the C restatement: L_i = Eq. 6 over
    knn_phase(x as binary32, g_index, K, r_max) at the first interaction."""
    cam = camera(cam_spec)
    ls = _lights(np.asarray(lights, np.float64).reshape(-1, 6))
    ph = tree.ph if tree is not None else np.ascontiguousarray(photons)
    src = PmSrc(_p(ph) if len(ph) else None, len(ph), tree.t if tree is not None else None, int(g_index),
                int(K), float(r_max))
    out = np.zeros((cam.height, cam.width, 3), np.float32)
    st = RenderStats()
    lib().or_render_photon_map(C.byref(scene.medium), ls, len(ls), C.byref(src), C.byref(cam),
                               C.byref(_rcfg(rc, cam, rect)), _p(out), C.byref(st))
    return out, {"samples": st.samples, "hits": st.hits}


# ------------------------------------------------------- photon tracing --


def hg_sample(g, w_in, u1, u2) -> np.ndarray:
    w = np.ascontiguousarray(w_in, dtype=np.float64)
    out = np.zeros(3)
    lib().or_hg_sample(float(g), _p(w), float(u1), float(u2), _p(out))
    return out


def emit_directions(light_pos, seed, stream, idx) -> np.ndarray:
    """emit_direction for photon streams make_rng(seed, stream, idx[i])."""
    P = np.ascontiguousarray(light_pos, dtype=np.float64)
    out = np.zeros((len(idx), 3))
    st = (C.c_uint64 * 2)()
    for i, j in enumerate(idx):
        lib().or_make_rng(st, seed, stream, int(j))
        lib().or_emit_direction(_p(P), st, _p(out[i]))
    return out


def trace_photons(scene: "OracleScene", lights, tc):
    """trace_photons (Alg. 1) on the C restatement.

    tc: object with n_total, phase_set, max_bounces, rr_start_bounce,
    rr_min_survival, rr_max_survival, seed.  Returns (photons, emitted[pairs],
    path_count[n_total]) with photons in the PHOTON_DTYPE layout (40 B)."""
    from paper_2304_07338_b200.scene import PHOTON_DTYPE
    gs = np.ascontiguousarray(tc.phase_set, dtype=np.float64)
    cfg = TraceCfg(int(tc.n_total), len(gs), _p(gs), tc.max_bounces, tc.rr_start_bounce,
                   float(tc.rr_min_survival), float(tc.rr_max_survival), int(tc.seed))
    L = _lights(np.asarray(lights, dtype=np.float64))
    emitted = np.zeros(max(1, len(lights) * len(gs)), np.uint64)
    paths = np.zeros(max(1, int(tc.n_total)), np.int32)
    cap = int(tc.n_total) * max(0, tc.max_bounces - 1) if tc.n_total < 200000 else int(tc.n_total) * 4
    while True:
        out = np.zeros(max(1, cap), dtype=PHOTON_DTYPE)
        n = lib().or_trace_photons(C.byref(scene.medium), L, len(lights), C.byref(cfg), _p(out), cap,
                                   _p(emitted), _p(paths))
        if n <= cap:
            break
        cap = n
    return out[:n].copy(), emitted[: len(lights) * len(gs)], paths[: int(tc.n_total)]


def ref_trace_photons(scene: "RefScene", lights, tc):
    """The pinned Alg. 1 composed from the reference's own primitives (ref_shim.cpp)."""
    from paper_2304_07338_b200.scene import make_photons
    L = np.ascontiguousarray(lights, dtype=np.float64).reshape(-1, 6)
    gs = np.ascontiguousarray(tc.phase_set, dtype=np.float64)
    cap = max(16, int(tc.n_total) * 4)
    while True:
        out9 = np.zeros((cap, 9), np.float32)
        og = np.zeros(cap, np.uint8)
        n = ref().ref_trace_photons(scene.h, _p(L), len(L), int(tc.n_total), len(gs), _p(gs),
                                    tc.max_bounces, tc.rr_start_bounce, float(tc.rr_min_survival),
                                    float(tc.rr_max_survival), int(tc.seed), _p(out9), _p(og), cap)
        if n <= cap:
            break
        cap = n
    return make_photons(out9[:n, 0:3], out9[:n, 3:6], out9[:n, 6:9], og[:n])
