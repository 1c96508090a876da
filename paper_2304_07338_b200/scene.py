"""Host-side scene data: volumes, transfer functions, lights, camera, photon maps.

Plain numpy plumbing around the device path.  Formats follow the reference:
  * volume raw + ".meta" sidecar  (proj/src/volume.cpp:79-131)
  * transfer-function text         (proj/src/volume.cpp:170-195)
  * photon map "PFPM"              (proj/include/pf/photon.hpp:59-64)
Synthetic generators are closed-form and RNG-free so the
oracle and the GPU always see the same bytes.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

# ------------------------------------------------------------ volumes -----


def synth_volume(kind: str, n: int | tuple[int, int, int]) -> np.ndarray:
    """Closed-form synthetic scalar volume, shape (nz, ny, nx) float32 (x fastest).

    kinds: "sphere_sinusoid" (SURVEY.md 8(d) scene A/B), "slab", "sphere"
    (SPEC.md:683-690), "constant:<v>".
    """
    nx, ny, nz = (n, n, n) if isinstance(n, int) else n
    out = np.empty((nz, ny, nx), dtype=np.float32)
    y, x = np.meshgrid((np.arange(ny) + 0.5) / ny, (np.arange(nx) + 0.5) / nx, indexing="ij")
    sx, sy = np.sin(18.0 * x), np.sin(18.0 * y)
    for k in range(nz):  # slab by slab: bounded host memory even at 1024^3
        z = (k + 0.5) / nz
        if kind == "sphere_sinusoid":
            r = np.sqrt((x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2)
            shell = np.clip(1.0 - r / 0.45, 0.0, 1.0)
            v = np.clip(shell * (0.55 + 0.45 * sx * sy * np.sin(18.0 * z)), 0.0, 1.0)
        elif kind == "slab":
            v = np.full(x.shape, 1.0 if 0.375 <= z <= 0.625 else 0.0)
        elif kind == "sphere":
            r = np.sqrt((x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2)
            v = (r <= 0.25).astype(np.float64)
        elif kind.startswith("constant:"):
            v = np.full(x.shape, float(kind.split(":")[1]))
        else:
            raise ValueError(f"unknown synthetic volume kind {kind!r}")
        out[k] = v
    return out


def validate_volume(v: np.ndarray) -> None:
    """VolumeGrid invariants (proj/src/volume.cpp:24-39)."""
    if v.ndim != 3 or min(v.shape) <= 0:
        raise ValueError("VolumeGrid: dims must be positive")
    if not np.all(np.isfinite(v)) or v.min() < 0.0 or v.max() > 1.0:
        raise ValueError("VolumeGrid: scalars must be finite and in [0,1]")


def save_volume(path: str | Path, v: np.ndarray) -> None:
    """raw binary32 + "<stem>.meta" (volume.cpp:120-131)."""
    path = Path(path)
    np.ascontiguousarray(v, dtype="<f4").tofile(path)
    nz, ny, nx = v.shape
    path.with_suffix(".meta").write_text(
        f"dims_x {nx}\ndims_y {ny}\ndims_z {nz}\nvalue_min 0\nvalue_max 1\n")


def load_volume(path: str | Path) -> np.ndarray:
    """VolumeGrid::load with range normalisation (volume.cpp:79-118)."""
    path = Path(path)
    meta = path.with_suffix(".meta")
    if not meta.exists():
        raise RuntimeError(f"VolumeGrid: cannot open {meta}")
    kv = {}
    for line in meta.read_text().splitlines():
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        if len(parts) >= 2:
            kv[parts[0]] = float(parts[1])
    for k in ("dims_x", "dims_y", "dims_z"):
        if k not in kv:
            raise RuntimeError(f"VolumeGrid: missing key '{k}' in metadata")
    nx, ny, nz = int(kv["dims_x"]), int(kv["dims_y"]), int(kv["dims_z"])
    data = np.fromfile(path, dtype="<f4")
    if data.size < nx * ny * nz:
        raise RuntimeError(f"VolumeGrid: {path} is shorter than dims imply")
    data = data[: nx * ny * nz].astype(np.float64)
    if not np.all(np.isfinite(data)):
        raise RuntimeError(f"VolumeGrid: non-finite scalar in {path}")
    vmin, vmax = kv.get("value_min", 0.0), kv.get("value_max", 1.0)
    rng = vmax - vmin
    n = (data - vmin) / rng if rng > 0 else np.zeros_like(data)
    return np.clip(n, 0.0, 1.0).astype(np.float32).reshape(nz, ny, nx)


# ---------------------------------------------------- transfer functions --


def validate_tf(points: np.ndarray) -> np.ndarray:
    """TransferFunction invariants (volume.cpp:136-149); returns (n,5) float64."""
    p = np.ascontiguousarray(points, dtype=np.float64)
    if p.ndim != 2 or p.shape[1] != 5 or p.shape[0] < 2:
        raise ValueError("TransferFunction: need at least two control points")
    if p[0, 0] != 0.0 or p[-1, 0] != 1.0:
        raise ValueError("TransferFunction: control points must span [0,1]")
    if not np.all((p[:, 1:] >= 0.0) & (p[:, 1:] <= 1.0)):
        raise ValueError("TransferFunction: channels must be in [0,1]")
    if np.any(np.diff(p[:, 0]) <= 0.0):
        raise ValueError("TransferFunction: positions must be strictly increasing")
    return p


def tf_scene_a() -> np.ndarray:
    """Scene A: sparse TF, ~11% hits, ~48 steps/sample."""
    return validate_tf([[0.0, 1.0, 1.0, 1.0, 0.0], [0.25, 0.9, 0.7, 0.5, 0.0],
                        [0.5, 0.8, 0.8, 0.9, 0.4], [1.0, 1.0, 1.0, 1.0, 1.0]])


def tf_scene_b() -> np.ndarray:
    """Scene B: denser TF, ~32% hits, ~20 steps/sample."""
    return validate_tf([[0.0, 1.0, 1.0, 1.0, 0.0], [0.02, 0.9, 0.6, 0.3, 0.02],
                        [0.5, 0.8, 0.8, 0.8, 0.3], [1.0, 1.0, 1.0, 1.0, 0.6]])


def save_tf(path: str | Path, p: np.ndarray) -> None:
    lines = ["# scalar r g b a"] + [" ".join(f"{v:.17g}" for v in row) for row in p]
    Path(path).write_text("\n".join(lines) + "\n")


def load_tf(path: str | Path) -> np.ndarray:
    rows = []
    for line in Path(path).read_text().splitlines():
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        if len(parts) >= 5:
            rows.append([float(v) for v in parts[:5]])
    return validate_tf(np.array(rows))


# ----------------------------------------------------- lights / camera ----


def default_lights() -> np.ndarray:
    """One point light at (2, 2.5, -1), intensity 1; n x 6."""
    return np.array([[2.0, 2.5, -1.0, 1.0, 1.0, 1.0]], dtype=np.float64)


@dataclass
class CameraSpec:
    """Pinhole camera."""
    width: int = 1920
    height: int = 1080
    position: tuple = (0.5, 0.5, -0.9)
    look_at: tuple = (0.5, 0.5, 0.5)
    up: tuple = (0.0, 1.0, 0.0)
    vfov_deg: float = 40.0


# ---------------------------------------------------------- photon map ----

PHOTON_DTYPE = np.dtype([("position", "<f4", 3), ("direction", "<f4", 3), ("power", "<f4", 3),
                         ("g_index", "u1"), ("pad_", "u1", 3)], align=False)
assert PHOTON_DTYPE.itemsize == 40


def make_photons(pos, dirs, power, g_index) -> np.ndarray:
    n = len(pos)
    a = np.zeros(n, dtype=PHOTON_DTYPE)
    a["position"] = pos
    a["direction"] = dirs
    a["power"] = power
    a["g_index"] = g_index
    return a


def synth_photons(n: int, n_phases: int = 3, seed: int = 0, clustered: bool = False) -> np.ndarray:
    """Synthetic photon map for the KNN benchmark."""
    r = np.random.default_rng(seed)
    if clustered:
        centers = r.random((64, 3))
        pos = centers[r.integers(0, 64, n)] + 0.05 * r.standard_normal((n, 3))
        pos = np.clip(pos, 0.0, 1.0)
    else:
        pos = r.random((n, 3))
    d = r.standard_normal((n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return make_photons(pos.astype(np.float32), d.astype(np.float32),
                        r.random((n, 3)).astype(np.float32), r.integers(0, n_phases, n))


@dataclass
class PhotonMapFile:
    photons: np.ndarray
    phase_set: list = field(default_factory=lambda: [-0.75, 0.0, 0.75])


_REC = np.dtype([("position", "<f4", 3), ("direction", "<f4", 3), ("power", "<f4", 3),
                 ("g_index", "u1")], align=False)
assert _REC.itemsize == 37


def save_photon_map(path: str | Path, photons: np.ndarray, phase_set) -> None:
    """PFPM: magic, u32 version, u64 count, u32 |G|, f64 g[], 37-B records."""
    rec = np.zeros(len(photons), dtype=_REC)
    for k in ("position", "direction", "power", "g_index"):
        rec[k] = photons[k]
    with open(path, "wb") as f:
        f.write(b"PFPM")
        f.write(struct.pack("<IQI", 1, len(photons), len(phase_set)))
        f.write(np.asarray(phase_set, dtype="<f8").tobytes())
        f.write(rec.tobytes())


def load_photon_map(path: str | Path) -> PhotonMapFile:
    raw = Path(path).read_bytes()
    if raw[:4] != b"PFPM":
        raise RuntimeError(f"{path}: not a PFPM photon map")
    ver, count, ng = struct.unpack_from("<IQI", raw, 4)
    if ver != 1:
        raise RuntimeError(f"{path}: unsupported PFPM version {ver}")
    off = 4 + 16
    phase = np.frombuffer(raw, dtype="<f8", count=ng, offset=off).tolist()
    off += 8 * ng
    if len(raw) - off < 37 * count:
        raise RuntimeError(f"{path}: truncated photon records")
    rec = np.frombuffer(raw, dtype=_REC, count=count, offset=off)
    return PhotonMapFile(make_photons(rec["position"], rec["direction"], rec["power"],
                                      rec["g_index"]), phase)
