"""Pin the CPU oracle against the reference's known answers.

Golden vectors: SURVEY.md Appendix A (computed with the reference's own
headers) and the SPEC's [TRIVIAL]/[DERIVED]/[PAPER] examples.
"""
import ctypes as C
import math

import numpy as np
import pytest

CAM, NEE, TEST = 3, 4, 8


def _draw_u32(o, seed, stream, index, n):
    r = (C.c_uint64 * 2)()
    o.lib().or_make_rng(r, seed, stream, index)
    return [o.lib().or_next_u32(r) for _ in range(n)], r


def test_rng_known_answers(oracle):
    # make_rng(0, Test, 0) -> 3 x next_u32, then next_double
    u, r = _draw_u32(oracle, 0, TEST, 0, 3)
    assert u == [3238339626, 1236702983, 2886652367]
    assert oracle.lib().or_next_double(r) == 0.86165437803801603
    # make_rng(7, CameraSample, 12345) -> next_double x 2
    r = (C.c_uint64 * 2)()
    oracle.lib().or_make_rng(r, 7, CAM, 12345)
    assert oracle.lib().or_next_double(r) == 0.98065389215791599
    assert oracle.lib().or_next_double(r) == 0.7036551539365844
    # make_rng(1, Nee, 0) -> next_u64 = 0x65d8e7f145f69684 (hi word first)
    u, _ = _draw_u32(oracle, 1, NEE, 0, 2)
    assert (u[0] << 32) | u[1] == 0x65D8E7F145F69684
    assert oracle.lib().or_splitmix64(0) == 0xE220A8397B1DCDAF


def test_hg_eval_known_answers(oracle):
    L = oracle.lib()
    assert abs(L.or_hg_eval(0.0, 0.3) - 1 / (4 * math.pi)) < 1e-15
    assert abs(L.or_hg_eval(0.5, 1.0) - 6 / (4 * math.pi)) < 1e-12
    for g in (-0.9, -0.35, 0.5, 0.75):                                      # symmetry
        for c in (-1.0, -0.2, 0.4, 1.0):
            assert abs(L.or_hg_eval(g, c) - L.or_hg_eval(-g, -c)) < 1e-12


def test_hg_normalisation(oracle):
    # SPEC phase invariant: 2*pi * int_{-1}^{1} hg dc == 1 within 1e-4
    c = np.linspace(-1, 1, 20001)
    for g in (-0.9, -0.75, -0.35, 0.0, 0.35, 0.5, 0.75, 0.9):
        v = np.array([oracle.lib().or_hg_eval(g, x) for x in c])
        assert abs(2 * math.pi * np.trapezoid(v, c) - 1.0) < 1e-4


def test_estimator_known_answers(oracle):
    L = oracle.lib()
    ph = np.zeros(1, dtype=np.dtype([("pos", "<f4", 3), ("dir", "<f4", 3), ("power", "<f4", 3),
                                     ("g", "u1"), ("pad", "u1", 3)]))
    ph["dir"] = [0, 0, 1]
    ph["power"] = [1, 1, 1]
    ids = np.zeros(1, np.uint32)
    d2 = np.array([0.25], np.float32)          # r = 0.5
    w = np.array([0.0, 0.0, 1.0])
    out = np.zeros(3)
    L.or_estimate_radiance(ph.ctypes.data, ids.ctypes.data, d2.ctypes.data, 1, w.ctypes.data, 0.0,
                           out.ctypes.data)
    assert np.allclose(out, 0.151981775, atol=1e-9)
    L.or_estimate_radiance(ph.ctypes.data, ids.ctypes.data, d2.ctypes.data, 0, w.ctypes.data, 0.0,
                           out.ctypes.data)
    assert np.all(out == 0.0)                                               # empty -> 0
    d2[0] = 0.0
    L.or_estimate_radiance(ph.ctypes.data, ids.ctypes.data, d2.ctypes.data, 1, w.ctypes.data, 0.0,
                           out.ctypes.data)
    assert np.all(out == 0.0)                                               # r < 1e-6 guard
    # Eq. 7 / Eq. 8
    assert L.or_encode_log(1.0, 5.0) == 0.0
    assert L.or_encode_log(0.0, 5.0) == 1.0
    assert abs(L.or_encode_log(1e-2, 4.0) - 0.5) < 1e-15
    assert L.or_encode_log(3.0, 5.0) == 0.0                                 # L > 1 clamp
    assert L.or_decode_log(0.0, 5.0) == 1.0
    assert abs(L.or_decode_log(1.0, 4.0) - 1e-4) < 1e-19
    for v in (1e-1, 1e-2, 1e-3):
        assert abs(L.or_decode_log(L.or_encode_log(v, 5.0), 5.0) / v - 1) < 1e-12


def test_schedule_radius(oracle):
    ends = np.array([0.36, 0.63, 0.90, 1.0])
    radii = np.array([0.25, 0.50, 2.50, 5.0])
    f = oracle.lib().or_schedule_radius
    assert f(ends.ctypes.data, radii.ctypes.data, 4, 0, 3000) == 0.25
    assert f(ends.ctypes.data, radii.ctypes.data, 4, 1080, 3000) == 0.50
    assert f(ends.ctypes.data, radii.ctypes.data, 4, 2950, 3000) == 5.0
    from paper_2304_07338_b200 import schedule_radius
    for s in range(0, 3000, 7):
        assert schedule_radius(ends, radii, s, 3000) == f(ends.ctypes.data, radii.ctypes.data, 4,
                                                          s, 3000)


def test_trilinear_known_answers(oracle):
    vol = np.array([0, 1, 1, 0, 1, 0, 0, 1], np.float32).reshape(2, 2, 2)
    tf = np.array([[0, 1, 1, 1, 1], [1, 1, 1, 1, 1]], np.float64)
    sc = oracle.OracleScene(vol, tf)
    assert sc.sample([0.5, 0.5, 0.5]) == 0.5
    assert sc.sample([0.25, 0.25, 0.25]) == 0.0                             # voxel centre
    assert sc.sample([0.75, 0.25, 0.25]) == 1.0
    cst = oracle.OracleScene(np.full((4, 4, 4), 0.5, np.float32), tf)
    for p in ([0.1, 0.2, 0.3], [0.9, 0.5, 0.0], [1.2, -0.1, 0.5]):
        assert cst.sample(p) == 0.5                                         # constant field


def test_transmittance_beer_lambert_golden(oracle):
    # homogeneous sigma = 2, length 1, 1e5 trials, make_rng(42, Test, 0) -> 0.13358
    vol = np.full((4, 4, 4), 1.0, np.float32)
    tf = np.array([[0, 1, 1, 1, 1], [1, 1, 1, 1, 1]], np.float64)
    sc = oracle.OracleScene(vol, tf, density_scale=2.0)
    T = sc.transmittance([[0.0, 0.5, 0.5]], [[1.0, 0.5, 0.5]], 42, TEST, [0], n_trials=100000)
    assert T[0] == 0.13358
    assert abs(T[0] - math.exp(-2)) / math.exp(-2) < 0.02


def test_vacuum(oracle):
    vol = np.zeros((8, 8, 8), np.float32)
    tf = np.array([[0, 1, 1, 1, 0], [1, 1, 1, 1, 1]], np.float64)
    sc = oracle.OracleScene(vol, tf)
    assert sc.sigma_max == 0.0
    n = 100
    o = np.tile([0.5, 0.5, -1.0], (n, 1))
    d = np.tile([0.0, 0.0, 1.0], (n, 1))
    hit, _, _ = sc.delta_track(o, d, np.zeros(n), np.full(n, np.inf), 0, CAM, np.arange(n))
    assert not hit.any()
    T = sc.transmittance(o, o + 2 * d, 0, NEE, np.arange(n))
    assert np.all(T == 1.0)


def test_mean_free_path(oracle):
    # homogeneous sigma = 5: mean free flight 1/sigma within 2%; KS
    vol = np.full((4, 4, 4), 1.0, np.float32)
    tf = np.array([[0, 1, 1, 1, 1], [1, 1, 1, 1, 1]], np.float64)
    sc = oracle.OracleScene(vol, tf, density_scale=5.0)
    n = 100000
    o = np.tile([0.5, 0.5, 0.0], (n, 1))
    d = np.tile([0.0, 0.0, 1.0], (n, 1))
    hit, pos, _ = sc.delta_track(o, d, np.zeros(n), np.full(n, 1e9), 9, TEST, np.arange(n))
    # flights past z = 1 leave the box; compare the truncated exponential
    t = pos[hit == 1, 2]
    p_exit = math.exp(-5.0)
    assert abs((1 - hit.mean()) - p_exit) < 3 * math.sqrt(p_exit / n) + 1e-3
    mean_trunc = (1 / 5.0) - math.exp(-5.0) / (1 - math.exp(-5.0))
    assert abs(t.mean() - mean_trunc) / mean_trunc < 0.02
    from scipy import stats
    cdf = lambda x: (1 - np.exp(-5.0 * x)) / (1 - math.exp(-5.0))  # noqa: E731
    assert stats.kstest(t, cdf).pvalue > 0.01


def test_photon_map_brute_force_edge_cases(oracle):
    from paper_2304_07338_b200.scene import make_photons
    ph = make_photons(np.array([[0.5, 0.5, 0.5]], np.float32), np.array([[0, 0, 1]], np.float32),
                      np.ones((1, 3), np.float32), np.array([1]))
    ids, d2 = oracle.knn_brute(ph, [0.5, 0.5, 0.5], 1, 1)
    assert list(ids) == [0] and d2[0] == 0.0
    ids, _ = oracle.knn_brute(ph, [0.5, 0.5, 0.5], 0, 4)
    assert len(ids) == 0                                                    # other phase
    empty = make_photons(np.zeros((0, 3), np.float32), np.zeros((0, 3), np.float32),
                         np.zeros((0, 3), np.float32), np.zeros(0))
    t = oracle.KdTree(empty)
    ids, _ = t.knn([0.1, 0.2, 0.3], 0, 8)
    assert len(ids) == 0
