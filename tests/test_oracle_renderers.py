"""The comparison renderers of the SPEC's render module on the CPU oracle.

render_path_traced and render_photon_map
have no reference code; their restatements in oracle/pf_oracle.c are pinned
  * against the reference's OWN primitives: ref_shim.cpp composes the same
    path tracer from pf::delta_track / pf::transmittance / pf::hg_sample /
    pf::make_rng -> bit-identical frames;
  * against an independent single-scatter quadrature (the SPEC's own oracle
    for render_path_traced);
  * against the SPEC's examples (alpha == 0 -> background, empty map ->
    direct light only, neural vs photon-map differ only through L_i).
"""
from types import SimpleNamespace

import numpy as np
import pytest

from paper_2304_07338_b200 import PathTraceConfig, RenderConfig
from paper_2304_07338_b200.scene import CameraSpec, default_lights, synth_photons, synth_volume, tf_scene_b


def _pt(mb=16):
    return PathTraceConfig(max_bounces=mb)


@pytest.fixture(scope="module")
def scene(oracle):
    vol = synth_volume("sphere_sinusoid", 32)
    return vol, oracle.OracleScene(vol, tf_scene_b())


@pytest.mark.parametrize("trials", [1, 2])
def test_path_traced_restatement_matches_reference_primitives(ref_oracle, scene, trials):
    vol, mine = scene
    ref = ref_oracle.RefScene(vol, tf_scene_b())
    cam = CameraSpec(width=40, height=32)
    # w_d = 0 isolates the continuation's L_i
    for w_d in (0.0, 1.0):
        rc = RenderConfig(spp=2, g=0.3, seed=11, w_d=w_d, background=(0.1, 0.2, 0.3), mode="parity",
                          nee_trials=trials)
        a, s1 = ref_oracle.render_path_traced(mine, default_lights(), cam, rc, _pt())
        b, s2 = ref_oracle.ref_render_path_traced(ref, default_lights(), cam, rc, _pt(), workers=3)
        assert s1["hits"] == s2["hits"] > 100
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert np.count_nonzero(a - 0.0) > 0


def test_path_traced_one_bounce_is_render_neural_without_field(oracle, scene):
    _, mine = scene
    cam = CameraSpec(width=32, height=24)
    rc = RenderConfig(spp=2, g=-0.4, seed=5, mode="parity", use_field=False, background=(0.2, 0.1, 0.0))
    a, _ = oracle.render_path_traced(mine, default_lights(), cam, rc, _pt(1))
    b, _ = oracle.render_neural(mine, default_lights(), None, None, cam, rc)
    assert np.array_equal(a, b)


def test_path_traced_indirect_grows_with_bounces(oracle, scene):
    """More vertices add (non-negative) in-scattered light; max_bounces beyond the
    roulette horizon changes almost nothing."""
    _, mine = scene
    cam = CameraSpec(width=24, height=24)
    rc = RenderConfig(spp=8, g=0.0, seed=3, w_d=0.0, mode="parity")
    means = [oracle.render_path_traced(mine, default_lights(), cam, rc, _pt(mb))[0].mean() for mb in (1, 2, 4, 16)]
    assert means[0] == 0.0
    assert means[1] > 0.0 and means[2] >= means[1] * 0.99 and means[3] >= means[2] * 0.99


def test_zero_alpha_volume_is_background_for_all_renderers(oracle):
    """alpha == 0 -> every pixel equals the background exactly."""
    vol = synth_volume("sphere_sinusoid", 16)
    tf = np.array([[0.0, 1, 1, 1, 0.0], [1.0, 1, 1, 1, 0.0]])
    osc = oracle.OracleScene(vol, tf)
    cam = CameraSpec(width=16, height=12)
    rc = RenderConfig(spp=2, g=0.0, seed=1, mode="parity", background=(0.25, 0.5, 0.75), use_field=False)
    bg = np.broadcast_to(np.float32([0.25, 0.5, 0.75]), (12, 16, 3))
    assert np.array_equal(oracle.render_path_traced(osc, default_lights(), cam, rc, _pt())[0], bg)
    ph = synth_photons(1000, 3, seed=1)
    assert np.array_equal(oracle.render_photon_map(osc, default_lights(), ph, 1, 16, np.inf, cam, rc)[0], bg)
    assert np.array_equal(oracle.render_neural(osc, default_lights(), None, None, cam, rc)[0], bg)


def test_single_scatter_quadrature(oracle):
    """homogeneous medium, max_bounces = 1 -> the mean image matches an
    independent single-scatter quadrature within 3%."""
    n = 8
    vol = np.full((n, n, n), 0.5, np.float32)
    sig = 2.0
    tf = np.array([[0.0, 1, 1, 1, sig / 100.0], [1.0, 1, 1, 1, sig / 100.0]])
    osc = oracle.OracleScene(vol, tf)
    light = np.array([[0.5, 1.6, 0.5, 1.0, 1.0, 1.0]])
    g = 0.3
    cam = CameraSpec(width=8, height=8, position=(0.5, 0.5, -1.2), look_at=(0.5, 0.5, 0.5), vfov_deg=40.0)
    rc = RenderConfig(spp=4000, g=g, seed=9, mode="parity", use_field=False)
    img, _ = oracle.render_path_traced(osc, light, cam, rc, _pt(1))

    # quadrature: E[sample] = int_0^{t1} sig e^{-sig t} L_d(x(t)) dt over the pixel footprint
    c = oracle.camera(cam)
    P = light[0, :3]
    f, r, u = (np.array(getattr(c, k)) for k in ("forward", "right", "up"))
    o = np.array(c.origin)
    js = (np.arange(8) + 0.5) / 8
    tq = None
    est = np.zeros((8, 8))
    for py in range(8):
        for px in range(8):
            acc = 0.0
            for ju in js:
                for jv in js:
                    sx = 2 * (px + ju) / 8 - 1
                    sy = 1 - 2 * (py + jv) / 8
                    d = f + r * sx + u * sy
                    d /= np.linalg.norm(d)
                    with np.errstate(divide="ignore"):
                        inv = 1.0 / d
                    t_a = (0.0 - o) * inv
                    t_b = (1.0 - o) * inv
                    t0 = max(0.0, np.max(np.minimum(t_a, t_b)))
                    t1 = np.min(np.maximum(t_a, t_b))
                    if t1 <= t0:
                        continue
                    m = 400
                    tq = t0 + (np.arange(m) + 0.5) * (t1 - t0) / m
                    x = o + tq[:, None] * d
                    v = x - P
                    dist = np.linalg.norm(v, axis=1)
                    din = v / dist[:, None]
                    # path length of x -> P inside the unit box (P is outside, above +y)
                    ty = (1.0 - x[:, 1]) / (-din[:, 1])  # din points from P to x: toward -y
                    inside = np.minimum(ty, dist)
                    cosang = din @ (-d)
                    hg = (1 - g * g) / (4 * np.pi * (1 + g * g - 2 * g * cosang) ** 1.5)
                    Ld = hg * np.exp(-sig * inside) / dist ** 2
                    acc += np.sum(sig * np.exp(-sig * (tq - t0)) * Ld) * (t1 - t0) / m
            est[py, px] = acc / 64
    mc = img[..., 0].astype(np.float64)
    print("mc mean", mc.mean(), "quadrature", est.mean())
    assert abs(mc.mean() - est.mean()) / est.mean() < 0.03


def test_photon_map_render_kdtree_equals_brute_force(oracle, scene):
    _, mine = scene
    ph = synth_photons(3000, 3, seed=2)
    ph["power"] *= 1e-3
    cam = CameraSpec(width=24, height=16)
    rc = RenderConfig(spp=1, g=0.0, seed=8, mode="parity")
    tree = oracle.KdTree(ph)
    a, _ = oracle.render_photon_map(mine, default_lights(), ph, 1, 32, 0.3, cam, rc, tree=tree)
    b, _ = oracle.render_photon_map(mine, default_lights(), ph, 1, 32, 0.3, cam, rc)
    assert np.array_equal(a, b)
    # neural vs photon-map backends differ only through L_i
    c, _ = oracle.render_neural(mine, default_lights(), None, None, cam,
                                RenderConfig(spp=1, g=0.0, seed=8, mode="parity", use_field=False))
    d, _ = oracle.render_photon_map(mine, default_lights(), ph, 1, 32, 0.3, cam,
                                    RenderConfig(spp=1, g=0.0, seed=8, mode="parity", w_i=0.0))
    assert np.array_equal(c, d)
    assert not np.array_equal(a, c)


def test_photon_map_render_empty_map_is_direct_light(oracle, scene):
    """empty map -> the direct-illumination-only image."""
    _, mine = scene
    cam = CameraSpec(width=16, height=16)
    rc = RenderConfig(spp=2, g=0.75, seed=4, mode="parity")
    empty = synth_photons(1, 3, seed=0)[:0]
    a, _ = oracle.render_photon_map(mine, default_lights(), empty, 2, 16, np.inf, cam, rc)
    b, _ = oracle.render_neural(mine, default_lights(), None, None, cam,
                                RenderConfig(spp=2, g=0.75, seed=4, mode="parity", use_field=False))
    assert np.array_equal(a, b)
