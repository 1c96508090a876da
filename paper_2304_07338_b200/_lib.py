"""ctypes binding of the C ABI in include/pf_gpu.h.

The shared library is built in-tree (paper_2304_07338_b200/libpfgpu.so,
see build.py).  There is no fallback: if it is missing or fails to load the
import of any GPU entry point raises -- the product path never silently
degrades to a CPU implementation.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# PF_LIBPFGPU: load another in-tree build of the same library (A/B of kernel
# variants in tools/); the default is the package's own libpfgpu.so.
LIB_PATH = Path(os.environ.get("PF_LIBPFGPU") or Path(__file__).resolve().parent / "libpfgpu.so")

PF_OK, PF_ERR_INVALID, PF_ERR_RUNTIME = 0, 1, 2
PF_MODE_PARITY, PF_MODE_FAST = 0, 1

# pf::Stream (proj/include/pf/rng.hpp:62-71)
STREAM = {"trace": 1, "train": 2, "camera": 3, "nee": 4, "pathtrace": 5, "fieldinit": 6,
          "synth": 7, "test": 8}


class HashGridDesc(C.Structure):
    _fields_ = [("dims", C.c_int), ("levels", C.c_int), ("features", C.c_int),
                ("base_res", C.c_int), ("growth", C.c_double), ("log2_table", C.c_int)]


class FieldDesc(C.Structure):
    _fields_ = [("pos", HashGridDesc), ("dir", HashGridDesc), ("hidden_layers", C.c_int),
                ("width", C.c_int), ("psi", C.c_double)]


class Camera(C.Structure):
    _fields_ = [("origin", C.c_double * 3), ("forward", C.c_double * 3),
                ("right", C.c_double * 3), ("up", C.c_double * 3),
                ("width", C.c_int), ("height", C.c_int)]


class RenderDesc(C.Structure):
    _fields_ = [("spp", C.c_int), ("g", C.c_double), ("seed", C.c_uint64),
                ("w_d", C.c_double), ("w_i", C.c_double), ("background", C.c_double * 3),
                ("mode", C.c_int), ("nee_trials", C.c_int), ("use_field", C.c_int),
                ("tile_w", C.c_int), ("tile_h", C.c_int), ("shard_index", C.c_int),
                ("shard_count", C.c_int)]


class RenderStats(C.Structure):
    _fields_ = [("samples", C.c_uint64), ("hits", C.c_uint64), ("primary_steps", C.c_uint64),
                ("shadow_steps", C.c_uint64), ("ms_trace", C.c_float), ("ms_field", C.c_float),
                ("ms_compose", C.c_float), ("kernel_launches", C.c_uint32),
                ("voxel_fetches", C.c_uint64)]


class Photon(C.Structure):
    """pf::Photon (proj/include/pf/photon.hpp:17-22), 40 bytes in memory."""
    _fields_ = [("position", C.c_float * 3), ("direction", C.c_float * 3),
                ("power", C.c_float * 3), ("g_index", C.c_uint8), ("pad_", C.c_uint8 * 3)]


assert C.sizeof(Photon) == 40


class TraceDesc(C.Structure):
    """pf::TraceConfig (proj/include/pf/photon.hpp:29-37)."""
    _fields_ = [("n_total", C.c_uint64), ("n_phases", C.c_int), ("phase_set", C.c_void_p),
                ("max_bounces", C.c_int), ("rr_start_bounce", C.c_int),
                ("rr_min_survival", C.c_double), ("rr_max_survival", C.c_double),
                ("seed", C.c_uint64)]

_P = C.c_void_p
class PathDesc(C.Structure):
    _fields_ = [("max_bounces", C.c_int), ("rr_start_bounce", C.c_int), ("rr_min_survival", C.c_double),
                ("rr_max_survival", C.c_double)]


_P_ = C.c_void_p


class AdamDesc(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("decay", C.c_double), ("decay_start", C.c_double), ("decay_interval", C.c_int),
                ("eps_rel", C.c_double)]


class TrainDesc(C.Structure):
    _fields_ = [("total_steps", C.c_uint64), ("batch", C.c_size_t), ("K", C.c_int), ("n_segments", C.c_int),
                ("seg_end", _P_), ("seg_radius", _P_), ("psi", C.c_double), ("seed", C.c_uint64),
                ("start_step", C.c_uint64), ("stop_step", C.c_uint64)]


_SIG = {
    "pf_last_error": (C.c_char_p, []),
    "pf_version": (C.c_char_p, []),
    "pf_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "pf_ctx_destroy": (None, [_P]),
    "pf_ctx_set_stream": (C.c_int, [_P, _P]),
    "pf_ctx_synchronize": (C.c_int, [_P]),
    "pf_ctx_set_timing": (C.c_int, [_P, C.c_int]),
    "pf_volume_upload": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, _P]),
    "pf_medium_set": (C.c_int, [_P, _P, C.c_int, C.c_double, C.c_double]),
    "pf_medium_sigma_max": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "pf_lights_set": (C.c_int, [_P, _P, C.c_int]),
    "pf_field_param_count": (C.c_int, [C.POINTER(FieldDesc), C.POINTER(C.c_size_t)]),
    "pf_field_init": (C.c_int, [C.POINTER(FieldDesc), C.c_uint64, C.c_double, C.c_double, _P]),
    "pf_field_load": (C.c_int, [_P, C.POINTER(FieldDesc), _P, C.c_size_t]),
    "pf_field_query": (C.c_int, [_P, C.c_size_t, _P, _P, _P, _P, C.c_int]),
    "pf_camera_make": (C.c_int, [_P, _P, _P, C.c_double, C.c_int, C.c_int, C.POINTER(Camera)]),
    "pf_render_neural": (C.c_int, [_P, C.POINTER(Camera), C.POINTER(RenderDesc), _P,
                                   C.POINTER(RenderStats)]),
    "pf_render_path_traced": (C.c_int, [_P, C.POINTER(Camera), C.POINTER(RenderDesc), C.POINTER(PathDesc),
                                        _P, C.POINTER(RenderStats)]),
    "pf_render_photon_map": (C.c_int, [_P, C.POINTER(Camera), C.POINTER(RenderDesc), C.c_int, C.c_float,
                                       _P, C.POINTER(RenderStats)]),
    "pf_tiles_count": (C.c_int, [C.POINTER(Camera), C.POINTER(RenderDesc), C.c_int,
                                 C.POINTER(C.c_int)]),
    "pf_tiles_pack": (C.c_int, [_P, C.POINTER(Camera), C.POINTER(RenderDesc), _P, _P]),
    "pf_tiles_unpack": (C.c_int, [_P, C.POINTER(Camera), C.POINTER(RenderDesc), _P, C.c_size_t,
                                  _P]),
    "pf_delta_track_batch": (C.c_int, [_P, C.c_size_t, _P, _P, _P, _P, C.c_uint64, C.c_uint64,
                                       _P, C.c_int, _P, _P, _P, _P]),
    "pf_transmittance_batch": (C.c_int, [_P, C.c_size_t, _P, _P, C.c_uint64, C.c_uint64, _P,
                                         C.c_int, _P]),
    "pf_transmittance_ratio_batch": (C.c_int, [_P, C.c_size_t, _P, _P, C.c_uint64, C.c_uint64,
                                               _P, C.c_int, _P]),
    "pf_rng_doubles": (C.c_int, [_P, C.c_size_t, C.c_uint64, C.c_uint64, _P, C.c_int, _P]),
    "pf_trace_photons": (C.c_int, [_P, _P, _P, _P]),
    "pf_trace_fetch": (C.c_int, [_P, _P, C.c_size_t]),
    "pf_trace_stats": (C.c_int, [_P, _P, _P, _P]),
    "pf_trace_path_counts": (C.c_int, [_P, _P, C.c_uint64]),
    "pf_knn_build_traced": (C.c_int, [_P, C.c_int, _P]),
    "pf_knn_build": (C.c_int, [_P, _P, C.c_size_t, C.c_int, _P]),
    "pf_knn_query": (C.c_int, [_P, C.c_size_t, _P, _P, C.c_int, C.c_float, _P, _P, _P]),
    "pf_knn_targets": (C.c_int, [_P, C.c_size_t, _P, _P, _P, C.c_int, C.c_float, C.c_double,
                                 _P, _P, _P, _P]),
    "pf_make_batch": (C.c_int, [_P, C.c_uint64, C.c_uint64, C.c_size_t, C.c_int, C.c_float,
                                C.c_double, _P, _P, _P, _P]),
    "pf_train_init": (C.c_int, [_P, C.POINTER(FieldDesc), _P, C.c_size_t, C.POINTER(AdamDesc)]),
    "pf_train_step": (C.c_int, [_P, C.c_size_t, _P, _P, _P, _P, C.c_uint64, C.c_uint64, _P]),
    "pf_train_grad": (C.c_int, [_P, C.c_size_t, _P, _P, _P, _P, _P, _P, _P]),
    "pf_train_counts": (C.c_int, [_P, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "pf_train_params": (C.c_int, [_P, _P, C.c_size_t]),
    "pf_train_commit": (C.c_int, [_P]),
    "pf_train": (C.c_int, [_P, C.POINTER(TrainDesc), _P, _P, _P, _P, _P]),
    "pf_train_state_get": (C.c_int, [_P, _P, _P, _P, C.c_size_t]),
    "pf_train_state_set": (C.c_int, [_P, _P, _P, _P, C.c_size_t]),
    "pf_ipc_frame_create": (C.c_int, [_P, C.c_size_t, C.POINTER(C.c_void_p), _P]),
    "pf_ipc_frame_open": (C.c_int, [_P, _P, C.POINTER(C.c_void_p)]),
    "pf_ipc_frame_release": (C.c_int, [_P, _P, C.c_int]),
    "pf_render_neural_async": (C.c_int, [_P, C.POINTER(Camera), C.POINTER(RenderDesc), _P]),
    "pf_frame_wait": (C.c_int, [_P, _P]),
    "pf_train_backward": (C.c_int, [_P, C.c_size_t, _P, _P, _P, _P, C.c_size_t, _P]),
    "pf_train_grad_buffers": (C.c_int, [_P, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.POINTER(C.c_void_p),
                                        C.POINTER(C.c_size_t), C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
    "pf_train_apply": (C.c_int, [_P, C.c_uint64, C.c_uint64]),
}
EXPORTS = tuple(_SIG)

_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    """Load libpfgpu.so (raises if it is absent -- no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2304_07338_b200.build` "
                               "(the photon-field path has no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIG.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    """Map a PF status to the reference's exception types."""
    if rc == PF_OK:
        return
    msg = lib().pf_last_error().decode()
    if rc == PF_ERR_INVALID:
        raise ValueError(msg)  # std::invalid_argument
    raise RuntimeError(msg)     # std::runtime_error / CUDA
