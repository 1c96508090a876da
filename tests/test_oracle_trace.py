"""Photon tracing (Alg. 1) on the CPU oracle: pinning + SPEC properties.

The reference declares trace_photons / emit_direction (photon.hpp:48-57) but
ships no definition, so the oracle's composition (oracle/pf_oracle.c
or_trace_photons) is pinned two ways:
  * against the same algorithm composed from the reference's OWN primitives
    (oracle/ref_shim.cpp ref_trace_photons: make_rng, delta_track, hg_sample,
    from_local_frame, Aabb::bounding_radius) -- bit-for-bit;
  * against SPEC.md:176-203's properties and examples.
"""
import math

import numpy as np
import pytest

from paper_2304_07338_b200.api import TraceConfig
from paper_2304_07338_b200.scene import (default_lights, load_photon_map, save_photon_map, synth_volume,
                                         tf_scene_a, tf_scene_b)

TRACE = 1


def _scene(oracle, kind="sphere_sinusoid", n=24, tf=None, density=100.0):
    return oracle.OracleScene(synth_volume(kind, n), tf_scene_b() if tf is None else tf, density)


def test_hg_sample_matches_reference_bitwise(ref_oracle):
    import ctypes as C
    o = ref_oracle
    r = np.random.default_rng(0)
    for _ in range(2000):
        g = float(r.choice([-0.999, -0.75, -1e-7, 0.0, 0.3, 0.75, 0.9995, r.uniform(-1, 1)]))
        w = r.standard_normal(3)
        w /= np.linalg.norm(w)
        if r.random() < 0.1:
            w = np.array([0.0, 0.0, float(r.choice([-1.0, 1.0]))])
        u1, u2 = float(r.random()), float(r.random())
        ref = (C.c_double * 3)()
        o.ref().ref_hg_sample(g, (C.c_double * 3)(*w), u1, u2, ref)
        assert list(o.hg_sample(g, w, u1, u2)) == list(ref)
        assert o.lib().or_hg_sample_cos(g, u1) == o.ref().ref_hg_sample_cos(g, u1)


@pytest.mark.parametrize("lights,tf", [
    (default_lights(), "b"),
    (np.array([[2.0, 2.5, -1.0, 1.0, 0.8, 0.6], [0.5, 0.5, 0.5, 0.3, 0.3, 0.3]]), "a"),  # 2nd light inside
])
def test_trace_matches_reference_composition(ref_oracle, lights, tf):
    o = ref_oracle
    vol = synth_volume("sphere_sinusoid", 20)
    tfp = tf_scene_b() if tf == "b" else tf_scene_a()
    sc = o.OracleScene(vol, tfp, 100.0)
    rs = o.RefScene(vol, tfp, 100.0)
    tc = TraceConfig(n_total=3000, seed=11)
    mine, emitted, paths = o.trace_photons(sc, lights, tc)
    ref = o.ref_trace_photons(rs, lights, tc)
    assert len(mine) > 500
    assert mine.tobytes() == ref.tobytes()
    assert emitted.sum() == tc.n_total and paths.sum() == len(mine)


def test_vacuum_gives_empty_map(oracle):
    sc = _scene(oracle, "constant:0.0", 8, tf=np.array([[0, 1, 1, 1, 0], [1, 1, 1, 1, 0.0]]))
    ph, emitted, _ = oracle.trace_photons(sc, default_lights(), TraceConfig(n_total=2000, seed=1))
    assert len(ph) == 0 and emitted.sum() == 2000


def test_stratification_tags_and_power(oracle):
    sc = _scene(oracle)
    lights = np.array([[2.0, 2.5, -1.0, 1.0, 0.5, 0.25], [-1.0, 0.5, 0.5, 2.0, 2.0, 2.0]])
    tc = TraceConfig(n_total=4001, seed=3)
    ph, emitted, paths = oracle.trace_photons(sc, lights, tc)
    assert emitted.max() - emitted.min() <= 1 and emitted.sum() == 4001   # SPEC: counts differ by <= 1
    assert set(np.unique(ph["g_index"])) <= {0, 1, 2}                      # g in G
    assert paths.max() <= tc.max_bounces - 1                                # no bounce-0 deposit
    assert np.all(np.isfinite(ph["power"])) and np.all(ph["power"] >= 0)
    # per-deposit power <= I / n_pair / rr_max (throughput <= 1, roulette-compensated)
    pair = np.repeat(np.arange(4001) % 6, paths)
    light = pair // 3
    bound = lights[light, 3:6] / emitted[pair][:, None] / tc.rr_max_survival
    assert np.all(ph["power"] <= bound * (1 + 1e-6))
    assert np.all((ph["position"] >= -1e-6) & (ph["position"] <= 1 + 1e-6))
    n = np.linalg.norm(ph["direction"].astype(np.float64), axis=1)
    assert np.all(np.abs(n - 1) < 1e-6)


def test_determinism(oracle):
    sc = _scene(oracle)
    tc = TraceConfig(n_total=1500, seed=9)
    a = oracle.trace_photons(sc, default_lights(), tc)[0]
    b = oracle.trace_photons(sc, default_lights(), tc)[0]
    assert a.tobytes() == b.tobytes()
    c = oracle.trace_photons(sc, default_lights(), TraceConfig(n_total=1500, seed=10))[0]
    assert a.tobytes() != c.tobytes()


def test_geometric_confinement_single_voxel(oracle):
    """one opaque voxel at the centre -> >= 95% of deposits
    within 2 voxel diagonals of it (1e5 photons)."""
    n = 16
    vol = np.zeros((n, n, n), np.float32)
    vol[n // 2, n // 2, n // 2] = 1.0
    tf = np.array([[0, 1, 1, 1, 0], [1, 1, 1, 1, 1.0]])
    sc = oracle.OracleScene(vol, tf, 400.0)
    ph, _, _ = oracle.trace_photons(sc, default_lights(), TraceConfig(n_total=100000, seed=2))
    assert len(ph) > 50
    c = np.array([(n // 2 + 0.5) / n] * 3)
    d = np.linalg.norm(ph["position"] - c, axis=1)
    assert np.mean(d <= 2 * math.sqrt(3) / n) >= 0.95


def test_emit_direction_far_light_cone(oracle):
    P = np.array([0.5, 0.5, 1000.0])
    w = oracle.emit_directions(P, 4, TRACE, np.arange(20000))
    assert np.all(np.abs(np.linalg.norm(w, axis=1) - 1) < 1e-12)
    axis = np.array([0, 0, -1.0])
    ang = np.arccos(np.clip(w @ axis, -1, 1))
    half = math.asin(0.5 * math.sqrt(3) / np.linalg.norm(P - 0.5))
    assert ang.max() <= half + 1e-9 and ang.max() > half * 0.99


def test_emit_direction_interior_light_uniform(oracle):
    w = oracle.emit_directions(np.array([0.5, 0.5, 0.5]), 4, TRACE, np.arange(100000))
    assert np.linalg.norm(w.mean(axis=0)) < 0.02
    assert np.all(np.abs(np.linalg.norm(w, axis=1) - 1) < 1e-12)


def test_every_emitted_ray_hits_bounding_sphere(oracle):
    P = np.array([2.0, 2.5, -1.0])
    w = oracle.emit_directions(P, 5, TRACE, np.arange(5000))
    v = np.array([0.5, 0.5, 0.5]) - P
    t = w @ v                                   # closest approach along each ray
    miss2 = (v ** 2).sum() - t ** 2
    assert np.all(t > 0) and np.all(miss2 <= 0.75 * (1 + 1e-12))


def test_trace_pfpm_roundtrip(oracle, tmp_path):
    sc = _scene(oracle)
    ph, _, _ = oracle.trace_photons(sc, default_lights(), TraceConfig(n_total=800, seed=4))
    save_photon_map(tmp_path / "m.pfpm", ph, [-0.75, 0.0, 0.75])
    back = load_photon_map(tmp_path / "m.pfpm")
    assert back.phase_set == [-0.75, 0.0, 0.75] and back.photons.tobytes() == ph.tobytes()
