"""Generate tests/golden/reference_c1.npz from the UNMODIFIED reference.

Run in the build container (needs /root/reference, compiled in place into
oracle/_ref by oracle/Makefile):  python tests/golden/make_golden.py
Everything stored here was produced by the reference's own code
(pf::make_rng / pf::delta_track / pf::transmittance, proj/src/volume.cpp,
proj/include/pf/rng.hpp) or by its parallel_chunks-driven render arm; the
volume itself is stored too so no regeneration can drift.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as o  # noqa: E402
from paper_2304_07338_b200 import RenderConfig  # noqa: E402
from paper_2304_07338_b200.scene import CameraSpec, default_lights, synth_volume, tf_scene_b  # noqa: E402

CAM, NEE, TEST = 3, 4, 8


def main():
    import ctypes as C
    R = o.ref()
    out = {}
    # 1. RNG streams
    seeds = np.array([0, 7, 1, 2024, 2 ** 63 + 5], np.uint64)
    idx = np.array([0, 1, 12345, 2 ** 40 + 3, 987654321], np.uint64)
    rng = np.zeros((len(seeds), 3, len(idx), 8))
    for a, sd in enumerate(seeds):
        for b, st in enumerate((CAM, NEE, TEST)):
            for c, ix in enumerate(idx):
                buf = (C.c_double * 8)()
                R.ref_rng_double(int(sd), st, int(ix), 8, buf)
                rng[a, b, c] = list(buf)
    out.update(rng_seeds=seeds, rng_idx=idx, rng_streams=np.array([CAM, NEE, TEST]), rng=rng)
    # 2. scene (stored)
    vol = synth_volume("sphere_sinusoid", 32)
    tf = tf_scene_b()
    sc = o.RefScene(vol, tf, 100.0)
    out.update(vol=vol, tf=tf, density=np.float64(100.0), sigma_max=np.float64(sc.sigma_max))
    # 3. delta_track
    r = np.random.default_rng(123)
    n = 4096
    org = np.tile([0.5, 0.5, -0.9], (n, 1))
    org[n // 2:] = r.uniform(-0.3, 1.3, (n // 2, 3))
    d = np.column_stack([r.uniform(-0.35, 0.35, n), r.uniform(-0.35, 0.35, n), np.ones(n)])
    d[n // 2:] = r.standard_normal((n // 2, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    tmin = np.zeros(n)
    tmax = np.full(n, np.inf)
    didx = np.arange(n, dtype=np.uint64) * 7 + 3
    hit, pos, rgba = sc.delta_track(org, d, tmin, tmax, 11, CAM, didx)
    out.update(dt_o=org, dt_d=d, dt_tmin=tmin, dt_tmax=tmax, dt_idx=didx, dt_seed=np.uint64(11),
               dt_hit=hit, dt_pos=pos, dt_rgba=rgba)
    # 4. transmittance
    m = 2048
    a = r.uniform(0.05, 0.95, (m, 3))
    b = np.tile([2.0, 2.5, -1.0], (m, 1))
    tidx = np.arange(m, dtype=np.uint64)
    out.update(tr_a=a, tr_b=b, tr_idx=tidx, tr_seed=np.uint64(5),
               tr_T1=sc.transmittance(a, b, 5, NEE, tidx, 1), tr_T3=sc.transmittance(a, b, 5, NEE, tidx, 3))
    # 5. render_neural, direct light only (reference delta_track/transmittance)
    cam = CameraSpec(48, 40)
    rc = RenderConfig(spp=2, g=0.3, seed=42, mode="parity", use_field=False, background=(0.05, 0.1, 0.2))
    img, st = o.ref_render_neural(sc, default_lights(), None, None, cam, rc, workers=4)
    out.update(img=img, img_hits=np.uint64(st["hits"]), img_spp=np.int32(2), img_g=np.float64(0.3),
               img_seed=np.uint64(42))
    np.savez_compressed(Path(__file__).with_name("reference_c1.npz"), **out)
    print({k: (v.shape if hasattr(v, "shape") else v) for k, v in out.items()})


if __name__ == "__main__":
    main()
