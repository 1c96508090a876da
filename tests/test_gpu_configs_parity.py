"""BASELINE configs 4 and 5 in PARITY mode (the bench headline's estimator)
against the UNMODIFIED reference (oracle/_ref: pf::delta_track /
pf::transmittance, proj/src/volume.cpp:204-256) on sampled full-width rows of
the full-size frames, plus the shard-union property at config 4.

Tolerance (as test_gpu_c2.py, direct light): hit counts within 1e-6 of the
samples + 2, <= 1e-3 of pixels differ at all and none by more than 1e-5
relative (the only source is a last-bit pf_log vs glibc log difference).
"""
import math

import numpy as np
import pytest

from paper_2304_07338_b200 import RenderConfig
from paper_2304_07338_b200.scene import CameraSpec, default_lights, synth_volume, tf_scene_a

pytestmark = pytest.mark.gpu


def _rows_match(ctx, ref_oracle, vol, tf, lights, cam, rc, rows):
    img = ctx.render_neural(cam, rc)
    sc = ref_oracle.RefScene(vol, tf, 100.0)
    diff_px, rel_max, n = 0, 0.0, 0
    for y in rows:
        ref, _ = ref_oracle.ref_render_neural(sc, lights, None, None, cam, rc, rect=(0, y, cam.width, y + 1))
        got, want = img[y].astype(np.float64), ref[y].astype(np.float64)
        d = np.any(got != want, axis=1)
        diff_px += int(d.sum())
        if d.any():
            rel_max = max(rel_max, float((np.abs(got - want) / np.maximum(np.abs(want), 1e-30))[d].max()))
        n += cam.width
    print(f"rows {rows}: {diff_px} of {n} pixels differ, max rel {rel_max:.3e}")
    assert diff_px <= max(2, 1e-3 * n)
    assert rel_max <= 1e-5
    return img


def test_config4_parity_rows_and_shard_union(ctx, ref_oracle):
    import torch
    vol = synth_volume("sphere_sinusoid", 512)
    tf, lights = tf_scene_a(), default_lights()
    ctx.upload_volume(vol)
    ctx.set_medium(tf, 100.0)
    ctx.set_lights(lights)
    spec = CameraSpec(3840, 2160)
    rc = RenderConfig(spp=16, seed=7, mode="parity", use_field=False)
    _rows_match(ctx, ref_oracle, vol, tf, lights, spec, rc, [300, 1080, 1500, 1999])
    cam = ctx.camera(spec)
    full = torch.zeros((2160, 3840, 3), device="cuda")
    ctx.render_neural(cam, rc, out=full)
    union = torch.zeros_like(full)
    for s in range(3):
        ctx.render_neural(cam, RenderConfig(spp=16, seed=7, mode="parity", use_field=False, shard_index=s,
                                            shard_count=3), out=union)
    ctx.synchronize()
    assert torch.equal(union, full)


def test_config5_parity_dynamic_frame_rows(ctx, ref_oracle):
    vol = synth_volume("sphere_sinusoid", 1024)
    ctx.upload_volume(vol)
    i = 3  # one frame of the per-frame TF + light animation (bench.dynamic_scene-like)
    tf = tf_scene_a()
    tf[:, 4] = np.clip(tf[:, 4] * (0.75 + 0.25 * math.cos(0.37 * i)), 0.0, 1.0)
    lights = default_lights()
    lights[0, 0], lights[0, 2] = 0.5 + 2.0 * math.cos(0.21 * i), 0.5 + 2.0 * math.sin(0.21 * i)
    ctx.set_medium(tf, 100.0)
    ctx.set_lights(lights)
    rc = RenderConfig(spp=8, seed=11, mode="parity", use_field=False)
    _rows_match(ctx, ref_oracle, vol, tf, lights, CameraSpec(1920, 1080), rc, [200, 540, 777])
