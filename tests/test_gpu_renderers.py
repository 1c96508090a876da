"""render_path_traced / render_photon_map on the GPU vs the oracle.

Tolerances (same reasoning as test_gpu_render.py):
  * PARITY: binary64 tracking with the reference's majorant and RNG
    consumption; frames equal the oracle's except where CUDA's log() rounds
    a last bit differently from glibc.  Path-traced frames: <= 1% of pixels
    differ by more than 1e-6 relative, frame RMSE <= 1e-3 x mean.  Photon-map
    frames (exact KNN + binary64 Eq. 6 in list order): <= 1e-3 of pixels.
  * max_bounces = 1 / w_i = 0 reproduce render_neural without a field (same
    program up to the first NEE): byte-for-byte in PARITY (--fmad=false);
    in FAST nvcc may contract the binary32 NEE arithmetic differently in the
    two kernels, so pixels agree to 1e-6 relative (last-ulp), same decisions.
  * FAST (binary32 DDA + ratio tracking): statistical -- frame means within
    3% of PARITY at high spp, per-pixel RMSE <= 1.3x the parity noise floor.
"""
import numpy as np
import pytest

from paper_2304_07338_b200 import PathTraceConfig, RenderConfig
from paper_2304_07338_b200.scene import CameraSpec, default_lights, synth_photons, synth_volume, tf_scene_b

pytestmark = pytest.mark.gpu

PHASES = [-0.75, 0.0, 0.75]


@pytest.fixture(scope="module")
def scene(ctx, oracle):
    vol = synth_volume("sphere_sinusoid", 48)
    tf = tf_scene_b()
    ctx.upload_volume(vol)
    ctx.set_medium(tf, 100.0)
    ctx.set_lights(default_lights())
    ph = synth_photons(20000, 3, seed=5)
    ph["power"] *= 1e-3
    ctx.knn_build(ph, PHASES)
    return ctx, oracle.OracleScene(vol, tf, 100.0), ph


def _rel_mismatch(a, b, rtol=1e-6):
    a = a.astype(np.float64)
    b = b.astype(np.float64)
    bad = np.abs(a - b) > rtol * np.maximum(np.abs(b), 1e-30)
    return np.count_nonzero(np.any(bad, axis=2))


@pytest.mark.parametrize("w_d", [0.0, 1.0])
def test_path_traced_parity_matches_oracle(scene, oracle, w_d):
    ctx, osc, _ = scene
    cam = CameraSpec(64, 48)
    rc = RenderConfig(spp=4, g=0.3, seed=21, w_d=w_d, mode="parity", background=(0.05, 0.1, 0.2))
    img, st = ctx.render_path_traced(cam, rc, PathTraceConfig(), stats=True)
    ref, ost = oracle.render_path_traced(osc, default_lights(), cam, rc, PathTraceConfig())
    n_bad = _rel_mismatch(img, ref)
    rmse = np.sqrt(np.mean((img.astype(np.float64) - ref) ** 2))
    print("pt parity: pixels >1e-6 rel", n_bad, "rmse", rmse, "mean", ref.mean(), "hits", st["hits"], ost["hits"])
    assert abs(st["hits"] - ost["hits"]) <= 2
    assert ref.mean() > 0
    assert n_bad <= 0.01 * 64 * 48
    assert rmse <= 1e-3 * ref.mean()


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_path_traced_one_bounce_is_render_neural(scene, mode):
    ctx, _, _ = scene
    cam = CameraSpec(80, 60)
    rc = RenderConfig(spp=2, g=-0.3, seed=3, mode=mode, use_field=False, background=(0.3, 0.2, 0.1))
    a = ctx.render_path_traced(cam, rc, PathTraceConfig(max_bounces=1))
    b = ctx.render_neural(cam, rc)
    if mode == "parity":
        assert np.array_equal(a, b)
    else:
        assert _rel_mismatch(a, b, 1e-6) == 0


def test_path_traced_fast_statistically_equal(scene):
    ctx, _, _ = scene
    cam = CameraSpec(48, 48)
    pt = PathTraceConfig()

    def r(mode, seed):
        return ctx.render_path_traced(cam, RenderConfig(spp=128, g=0.5, seed=seed, w_d=0.0, mode=mode), pt
                                      ).astype(np.float64)
    par, par2, fast = r("parity", 1), r("parity", 2), r("fast", 3)
    noise = np.sqrt(np.mean((par2 - par) ** 2))
    err = np.sqrt(np.mean((fast - par) ** 2))
    print("pt fast vs parity rmse", err, "noise", noise, "means", fast.mean(), par.mean(), par2.mean())
    assert abs(fast.mean() - par.mean()) / par.mean() < 0.03
    assert err < 1.3 * noise


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_path_traced_shard_invariance(scene, mode):
    ctx, _, _ = scene
    cam = CameraSpec(70, 45)
    import torch
    full = ctx.render_path_traced(cam, RenderConfig(spp=2, g=0.2, seed=9, mode=mode, tile=(16, 8)))
    parts = torch.zeros((45, 70, 3), dtype=torch.float32, device="cuda")
    for s in range(3):
        ctx.render_path_traced(cam, RenderConfig(spp=2, g=0.2, seed=9, mode=mode, tile=(16, 8), shard_index=s,
                                                 shard_count=3), out=parts)
    ctx.synchronize()
    assert np.array_equal(parts.cpu().numpy().view(np.uint32), full.view(np.uint32))


def test_path_traced_argument_errors(scene):
    ctx, _, _ = scene
    cam = CameraSpec(8, 8)
    with pytest.raises(ValueError, match="max_bounces"):
        ctx.render_path_traced(cam, RenderConfig(), PathTraceConfig(max_bounces=0))
    with pytest.raises(ValueError, match="rr_min"):
        ctx.render_path_traced(cam, RenderConfig(), PathTraceConfig(rr_min_survival=0.0))
    with pytest.raises(ValueError, match="spp"):
        ctx.render_path_traced(cam, RenderConfig(spp=0))


@pytest.mark.parametrize("K,r_max", [(32, float("inf")), (64, 0.08)])
def test_photon_map_parity_matches_oracle(scene, oracle, K, r_max):
    ctx, osc, ph = scene
    cam = CameraSpec(64, 48)
    rc = RenderConfig(spp=2, g=0.75, seed=17, mode="parity")
    img, st = ctx.render_photon_map(cam, rc, K=K, r_max=r_max, stats=True)
    tree = oracle.KdTree(ph)
    ref, ost = oracle.render_photon_map(osc, default_lights(), ph, 2, K, r_max, cam, rc, tree=tree)
    n_bad = _rel_mismatch(img, ref, 1e-12)
    print("pm parity: pixels differing", n_bad, "mean", ref.mean(), "hits", st["hits"], ost["hits"])
    assert abs(st["hits"] - ost["hits"]) <= 2
    assert n_bad <= max(3, 1e-3 * 64 * 48)


def test_photon_map_without_li_is_render_neural(scene):
    ctx, _, _ = scene
    cam = CameraSpec(40, 30)
    for mode in ("parity", "fast"):
        a = ctx.render_photon_map(cam, RenderConfig(spp=2, g=0.0, seed=4, mode=mode, w_i=0.0), K=16)
        b = ctx.render_neural(cam, RenderConfig(spp=2, g=0.0, seed=4, mode=mode, use_field=False))
        c = ctx.render_photon_map(cam, RenderConfig(spp=2, g=0.0, seed=4, mode=mode), K=16)
        assert np.array_equal(a, b)
        assert not np.array_equal(c, b)


def test_photon_map_fast_statistically_equal(scene):
    ctx, _, _ = scene
    cam = CameraSpec(48, 48)

    def r(mode, seed):
        return ctx.render_photon_map(cam, RenderConfig(spp=64, g=-0.75, seed=seed, w_d=0.0, mode=mode), K=64
                                     ).astype(np.float64)
    par, par2, fast = r("parity", 1), r("parity", 2), r("fast", 3)
    noise = np.sqrt(np.mean((par2 - par) ** 2))
    err = np.sqrt(np.mean((fast - par) ** 2))
    print("pm fast vs parity rmse", err, "noise", noise, "means", fast.mean(), par.mean())
    assert abs(fast.mean() - par.mean()) / par.mean() < 0.03
    assert err < 1.3 * noise


def test_photon_map_argument_errors(scene):
    ctx, _, _ = scene
    cam = CameraSpec(8, 8)
    with pytest.raises(ValueError, match="phase set"):
        ctx.render_photon_map(cam, RenderConfig(g=0.5), K=8)
    with pytest.raises(ValueError, match="K must"):
        ctx.render_photon_map(cam, RenderConfig(g=0.0), K=0)
    with pytest.raises(ValueError, match="r_max"):
        ctx.render_photon_map(cam, RenderConfig(g=0.0), K=8, r_max=0.0)


def test_zero_alpha_all_renderers_background(ctx):
    vol = synth_volume("sphere_sinusoid", 16)
    ctx.upload_volume(vol)
    ctx.set_medium(np.array([[0.0, 1, 1, 1, 0.0], [1.0, 1, 1, 1, 0.0]]), 100.0)
    ctx.set_lights(default_lights())
    ctx.knn_build(synth_photons(500, 3, seed=1), PHASES)
    cam = CameraSpec(20, 10)
    bg = np.broadcast_to(np.float32([0.25, 0.5, 0.75]), (10, 20, 3))
    for mode in ("parity", "fast"):
        rc = RenderConfig(spp=2, g=0.0, mode=mode, background=(0.25, 0.5, 0.75), use_field=False)
        assert np.array_equal(ctx.render_path_traced(cam, rc), bg)
        assert np.array_equal(ctx.render_photon_map(cam, rc, K=8), bg)
        assert np.array_equal(ctx.render_neural(cam, rc), bg)


def test_photon_map_empty_map_is_direct_light(ctx):
    vol = synth_volume("sphere_sinusoid", 24)
    ctx.upload_volume(vol)
    ctx.set_medium(tf_scene_b(), 100.0)
    ctx.set_lights(default_lights())
    ctx.knn_build(synth_photons(1, 3, seed=0)[:0], PHASES)
    cam = CameraSpec(24, 24)
    for mode in ("parity", "fast"):
        a = ctx.render_photon_map(cam, RenderConfig(spp=2, g=0.75, seed=4, mode=mode), K=16)
        b = ctx.render_neural(cam, RenderConfig(spp=2, g=0.75, seed=4, mode=mode, use_field=False))
        assert np.array_equal(a, b)


def test_two_lights_three_trials_parity(ctx, oracle):
    """The per-light NEE loop with n_trials > 1 (transmittance's trial loop,
    volume.cpp:240-255) in every renderer, against the oracle."""
    vol = synth_volume("sphere_sinusoid", 32)
    tf = tf_scene_b()
    lights = np.array([[2.0, 2.5, -1.0, 1.0, 0.8, 0.6], [-1.0, 0.5, 0.5, 0.3, 0.5, 1.0]])
    ctx.upload_volume(vol)
    ctx.set_medium(tf, 100.0)
    ctx.set_lights(lights)
    ph = synth_photons(8000, 3, seed=9)
    ph["power"] *= 1e-3
    ctx.knn_build(ph, PHASES)
    osc = oracle.OracleScene(vol, tf, 100.0)
    cam = CameraSpec(40, 30)
    rc = RenderConfig(spp=2, g=-0.75, seed=13, mode="parity", nee_trials=3, background=(0.1, 0.1, 0.1))
    pt = PathTraceConfig(max_bounces=6)
    got = ctx.render_path_traced(cam, rc, pt)
    ref, _ = oracle.render_path_traced(osc, lights, cam, rc, pt)
    assert _rel_mismatch(got, ref) <= 0.01 * 40 * 30
    got = ctx.render_photon_map(cam, rc, K=16, r_max=0.2)
    ref, _ = oracle.render_photon_map(osc, lights, ph, 0, 16, 0.2, cam, rc)
    assert _rel_mismatch(got, ref, 1e-12) <= 3
    rc2 = RenderConfig(spp=2, g=-0.75, seed=13, mode="parity", nee_trials=3, use_field=False)
    got = ctx.render_neural(cam, rc2)
    ref, _ = oracle.render_neural(osc, lights, None, None, cam, rc2)
    assert _rel_mismatch(got, ref, 1e-12) <= 3


def test_path_traced_noise_falls_with_spp(ctx):
    """pixel variance at 1 spp > at 64 spp (same scene, same pixels)."""
    ctx.upload_volume(synth_volume("sphere_sinusoid", 32))
    ctx.set_medium(tf_scene_b(), 100.0)
    ctx.set_lights(default_lights())
    cam = CameraSpec(32, 32)
    pt = PathTraceConfig(max_bounces=8)

    def var(spp):
        a, b = (ctx.render_path_traced(cam, RenderConfig(spp=spp, g=0.3, seed=s, mode="fast"), pt).astype(np.float64)
                for s in (1, 2))
        return np.mean((a - b) ** 2) / 2
    v1, v64 = var(1), var(64)
    print("pt pixel variance 1 spp", v1, "64 spp", v64)
    assert v1 > 8 * v64


def test_photon_map_consistency_with_photon_count(ctx):
    """more photons -> strictly lower MSE against a dense-map
    reference render (median over 3 seeds), with maps traced on the device."""
    from paper_2304_07338_b200 import TraceConfig
    ctx.upload_volume(synth_volume("sphere_sinusoid", 32))
    ctx.set_medium(tf_scene_b(), 100.0)
    ctx.set_lights(default_lights())
    cam = CameraSpec(48, 48)
    rc = RenderConfig(spp=16, g=0.0, seed=3, mode="fast", w_d=0.0)

    def render(n, seed):
        tc = TraceConfig(n_total=n, seed=seed)
        ctx.trace_photons(tc, device=True)
        ctx.knn_build_traced(tc.phase_set)
        return ctx.render_photon_map(cam, rc, K=64).astype(np.float64)
    ref = render(8_000_000, 99)
    med = [np.median([np.mean((render(n, s) - ref) ** 2) for s in range(3)]) for n in (10_000, 100_000, 1_000_000)]
    print("pm mse vs photon count", med)
    assert med[0] > med[1] > med[2]
