"""The C restatement (oracle/pf_oracle.c) vs the UNMODIFIED reference (oracle/_ref).

Bit-for-bit: both are binary64 x86 code compiled with -ffp-contract=off, and
the restatement follows volume.cpp / rng.hpp / math.hpp operation by operation.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2304_07338_b200.scene import CameraSpec, default_lights, synth_volume, tf_scene_a, tf_scene_b

CAM, NEE, TEST = 3, 4, 8


def _rays(n, seed=0):
    r = np.random.default_rng(seed)
    o = r.uniform(-0.5, 1.5, (n, 3))
    o[: n // 4] = r.uniform(0, 1, (n // 4, 3))               # interior origins
    d = r.standard_normal((n, 3))
    d[n // 4: n // 4 + 64, 0] = 0.0                           # axis-parallel (NaN slab terms)
    d[n // 4 + 64: n // 4 + 128, 1:] = 0.0
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o[n // 4 + 128: n // 4 + 160] = [0.0, 0.5, -1.0]          # face-grazing: x = 0 plane
    d[n // 4 + 128: n // 4 + 160] = [0.0, 0.0, 1.0]
    tmin = np.zeros(n)
    tmin[::7] = r.uniform(0, 0.5, len(tmin[::7]))
    tmax = np.full(n, np.inf)
    tmax[::5] = r.uniform(0.6, 3.0, len(tmax[::5]))
    return o, d, tmin, tmax


def test_rng_streams_bitwise(ref_oracle):
    o = ref_oracle
    for seed, stream, index in [(0, 8, 0), (7, 3, 12345), (1, 4, 0), (2**63 + 5, 2, 2**40 + 3)]:
        a = (C.c_uint32 * 9)()
        o.ref().ref_rng_u32(seed, stream, index, 9, a)
        r = (C.c_uint64 * 2)()
        o.lib().or_make_rng(r, seed, stream, index)
        assert [o.lib().or_next_u32(r) for _ in range(9)] == list(a)
    idx = np.arange(1000, dtype=np.uint64) * 977
    mine = np.zeros((1000, 6))
    o.lib().or_rng_doubles(5, 3, 1000, idx.ctypes.data, 6, mine.ctypes.data)
    for i in range(0, 1000, 37):
        ref = (C.c_double * 6)()
        o.ref().ref_rng_double(5, 3, int(idx[i]), 6, ref)
        assert list(mine[i]) == list(ref)


def test_phase_known_answers_reference(ref_oracle):
    R = ref_oracle.ref()
    # SURVEY App. A values produced by the reference itself
    assert R.ref_hg_sample_cos(0.75, 0.3) == 0.78125
    assert R.ref_hg_cdf(0.75, 0.78125) == 0.30000000000000004
    out = (C.c_double * 3)()
    R.ref_hg_sample(0.75, (C.c_double * 3)(0, 0, 1), 0.3, 0.6, out)
    assert list(out) == [-0.50500318143509981, -0.36690628809060721, 0.78125]
    for g in (-0.999, -0.5, 0.0, 0.2, 0.9, 1.5):
        for c in (-1.0, -0.3, 0.0, 0.7, 1.0):
            assert ref_oracle.lib().or_hg_eval(g, c) == R.ref_hg_eval(g, c)


def test_aabb_bitwise(ref_oracle):
    o, d, tmin, tmax = _rays(2000, 3)
    for i in range(2000):
        a0, a1, b0, b1 = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        ra = ref_oracle.ref().ref_aabb_intersect(o[i].ctypes.data, d[i].ctypes.data, tmin[i], tmax[i],
                                                C.byref(a0), C.byref(a1))
        rb = ref_oracle.lib().or_aabb_intersect(o[i].ctypes.data, d[i].ctypes.data, tmin[i], tmax[i],
                                               C.byref(b0), C.byref(b1))
        assert ra == rb
        if ra:
            assert (a0.value, a1.value) == (b0.value, b1.value)
    # face-grazing ray with dir.x = 0 at x = 0 is a hit, t0 = 1, t1 = 2
    a0, a1 = C.c_double(), C.c_double()
    assert ref_oracle.lib().or_aabb_intersect(np.array([0.0, 0.5, -1.0]).ctypes.data,
                                              np.array([0.0, 0.0, 1.0]).ctypes.data, 0.0, np.inf,
                                              C.byref(a0), C.byref(a1)) == 1
    assert (a0.value, a1.value) == (1.0, 2.0)


@pytest.mark.parametrize("tf", [tf_scene_a, tf_scene_b])
def test_medium_and_sampling_bitwise(ref_oracle, tf):
    vol = synth_volume("sphere_sinusoid", 24)
    mine = ref_oracle.OracleScene(vol, tf())
    ref = ref_oracle.RefScene(vol, tf())
    assert mine.sigma_max == ref.sigma_max
    r = np.random.default_rng(1)
    for p in r.uniform(-0.2, 1.2, (500, 3)):
        assert mine.sample(p) == ref_oracle.ref().ref_grid_sample(ref.h, p.ctypes.data)
    for s in np.concatenate([r.uniform(-0.5, 1.5, 200), tf()[:, 0]]):
        a, b = np.zeros(4), np.zeros(4)
        ref_oracle.lib().or_tf_classify(C.byref(mine.tfs), float(s), a.ctypes.data)
        ref_oracle.ref().ref_tf_classify(ref.h, float(s), b.ctypes.data)
        assert list(a) == list(b)


@pytest.mark.parametrize("tf", [tf_scene_a, tf_scene_b])
def test_delta_track_bitwise(ref_oracle, tf):
    vol = synth_volume("sphere_sinusoid", 32)
    mine = ref_oracle.OracleScene(vol, tf())
    ref = ref_oracle.RefScene(vol, tf())
    o, d, tmin, tmax = _rays(20000, 11)
    idx = np.arange(20000, dtype=np.uint64) * 3 + 1
    h1, p1, c1 = mine.delta_track(o, d, tmin, tmax, 77, CAM, idx)
    h2, p2, c2 = ref.delta_track(o, d, tmin, tmax, 77, CAM, idx)
    assert h1.sum() > 1000
    assert np.array_equal(h1, h2)
    assert np.array_equal(p1.view(np.uint64), p2.view(np.uint64))
    assert np.array_equal(c1.view(np.uint64), c2.view(np.uint64))


def test_delta_track_invalid_ray(ref_oracle):
    vol = synth_volume("sphere_sinusoid", 8)
    mine = ref_oracle.OracleScene(vol, tf_scene_b())
    ref = ref_oracle.RefScene(vol, tf_scene_b())
    for bad in ([np.nan, 0, 0], ):
        with pytest.raises(ValueError):
            mine.delta_track([bad], [[0, 0, 1]], [0.0], [np.inf], 0, CAM, [0])
        with pytest.raises(ValueError):
            ref.delta_track([bad], [[0, 0, 1]], [0.0], [np.inf], 0, CAM, [0])
    with pytest.raises(ValueError):   # t_min > t_max (volume.cpp:205-207)
        ref.delta_track([[0, 0, 0]], [[0, 0, 1]], [2.0], [1.0], 0, CAM, [0])


@pytest.mark.parametrize("n_trials", [1, 3])
def test_transmittance_bitwise(ref_oracle, n_trials):
    vol = synth_volume("sphere_sinusoid", 32)
    mine = ref_oracle.OracleScene(vol, tf_scene_a())
    ref = ref_oracle.RefScene(vol, tf_scene_a())
    r = np.random.default_rng(5)
    a = r.uniform(0, 1, (5000, 3))
    b = np.tile([2.0, 2.5, -1.0], (5000, 1))
    b[::9] = a[::9]                                      # zero-length segments -> 1.0
    idx = np.arange(5000, dtype=np.uint64)
    t1 = mine.transmittance(a, b, 3, NEE, idx, n_trials)
    t2 = ref.transmittance(a, b, 3, NEE, idx, n_trials)
    assert np.array_equal(t1, t2)
    assert 0.05 < t1.mean() < 0.95


def test_render_restatement_matches_reference_path(ref_oracle):
    """or_render_neural (C restatement) == reference delta_track/transmittance driver."""
    from paper_2304_07338_b200 import FieldConfig, RenderConfig
    vol = synth_volume("sphere_sinusoid", 32)
    fc = FieldConfig.desk()
    params = fc.init_params(seed=3, embed_scale=0.5, bias_scale=0.1)
    cam = CameraSpec(width=40, height=32)
    rc = RenderConfig(spp=2, g=0.3, seed=11, background=(0.1, 0.2, 0.3), mode="parity")
    mine = ref_oracle.OracleScene(vol, tf_scene_b())
    ref = ref_oracle.RefScene(vol, tf_scene_b())
    img1, st1 = ref_oracle.render_neural(mine, default_lights(), fc, params, cam, rc)
    img2, st2 = ref_oracle.ref_render_neural(ref, default_lights(), fc, params, cam, rc, workers=3)
    assert st1["hits"] == st2["hits"] > 100
    assert np.array_equal(img1.view(np.uint32), img2.view(np.uint32))
