"""Device photon tracer (Alg. 1, pf_trace_photons) vs the oracle.

Parity bar: records are produced per photon in (photon, bounce) order from
make_rng(seed, Trace, i).  The device computes the same binary64 operation
sequence (--fmad=false), but CUDA's log/sin/cos differ from glibc's in the
last ulp for a small fraction of arguments; a different last bit can (rarely)
flip a delta-tracking decision and send that photon down another path.  So:
  * >= 99% of photons produce byte-identical deposit records, and
  * the rest are statistically indistinguishable (deposit counts, power sums).
"""
import numpy as np
import pytest

from paper_2304_07338_b200.api import TraceConfig
from paper_2304_07338_b200.scene import default_lights, synth_volume, tf_scene_a, tf_scene_b

pytestmark = pytest.mark.gpu

LIGHTS2 = np.array([[2.0, 2.5, -1.0, 1.0, 0.8, 0.6], [0.5, 0.5, 0.5, 0.3, 0.3, 0.3]])


def _split(ph, counts):
    offs = np.concatenate([[0], np.cumsum(counts.astype(np.int64))])
    raw = ph.tobytes()
    return [raw[40 * offs[i]: 40 * offs[i + 1]] for i in range(len(counts))]


@pytest.mark.parametrize("tf,lights,n", [("b", default_lights(), 20000), ("a", LIGHTS2, 12000)])
def test_trace_matches_oracle(ctx, oracle, tf, lights, n):
    vol = synth_volume("sphere_sinusoid", 32)
    tfp = tf_scene_b() if tf == "b" else tf_scene_a()
    ctx.upload_volume(vol)
    ctx.set_medium(tfp, 100.0)
    ctx.set_lights(lights)
    tc = TraceConfig(n_total=n, seed=21)
    res = ctx.trace_photons(tc)
    counts = ctx.trace_path_counts(n)
    mine, emitted, paths = oracle.trace_photons(oracle.OracleScene(vol, tfp, 100.0), lights, tc)
    assert np.array_equal(res.emitted_per_pair, emitted)
    a, b = _split(res.photons, counts), _split(mine, paths)
    same = np.mean([x == y for x, y in zip(a, b)])
    print(f"identical photons {same:.5f}  deposits gpu {len(res.photons)} oracle {len(mine)}")
    assert same >= 0.99
    assert abs(len(res.photons) - len(mine)) <= max(10, 0.01 * len(mine))
    pg, po = res.photons["power"].astype(np.float64).sum(0), mine["power"].astype(np.float64).sum(0)
    assert np.all(np.abs(pg - po) <= 0.02 * po)


def test_trace_determinism_device_output_and_errors(ctx):
    import torch
    ctx.upload_volume(synth_volume("sphere_sinusoid", 32))
    ctx.set_medium(tf_scene_b(), 100.0)
    ctx.set_lights(default_lights())
    tc = TraceConfig(n_total=50000, seed=5)
    a = ctx.trace_photons(tc)
    b = ctx.trace_photons(tc, device=True)
    assert a.photons.tobytes() == b.photons.cpu().numpy().tobytes()
    assert np.all(a.photons["pad_"] == 0)
    with pytest.raises(ValueError):
        ctx.trace_photons(TraceConfig(n_total=10, phase_set=[]))
    with pytest.raises(ValueError):
        ctx.trace_photons(TraceConfig(n_total=10, phase_set=[0.5, 0.5]))
    with pytest.raises(ValueError):
        ctx.trace_photons(TraceConfig(n_total=10, phase_set=[1.5]))
    with pytest.raises(ValueError):
        ctx.trace_photons(TraceConfig(n_total=10, max_bounces=0))
    ctx.set_lights(np.zeros((0, 6)))
    with pytest.raises(ValueError):
        ctx.trace_photons(TraceConfig(n_total=10))
    ctx.set_lights(default_lights())
    z = ctx.trace_photons(TraceConfig(n_total=0))
    assert len(z.photons) == 0
    del torch


def test_trace_vacuum_empty(ctx):
    ctx.upload_volume(synth_volume("constant:0.0", 16))
    ctx.set_medium(np.array([[0, 1, 1, 1, 0], [1, 1, 1, 1, 0.0]]), 100.0)
    ctx.set_lights(default_lights())
    r = ctx.trace_photons(TraceConfig(n_total=100000, seed=1))
    assert len(r.photons) == 0 and r.emitted_per_pair.sum() == 100000


def test_trace_large_properties_and_knn_from_trace(ctx, oracle):
    """2M photons (the scale a training run uses): SPEC invariants at full size,
    plus KNN built straight from the resident trace == KNN built from a copy."""
    ctx.upload_volume(synth_volume("sphere_sinusoid", 128))
    ctx.set_medium(tf_scene_b(), 100.0)
    ctx.set_lights(LIGHTS2)
    ctx.set_timing(True)
    tc = TraceConfig(n_total=2_000_000, seed=8)
    res = ctx.trace_photons(tc)
    st = ctx.trace_stats()
    ctx.set_timing(False)
    ph = res.photons
    counts = ctx.trace_path_counts(tc.n_total)
    print(f"2M photons: {len(ph)} deposits, trace {st['ms_trace']:.2f} ms, compact {st['ms_compact']:.2f} ms, "
          f"{st['tentative_collisions'] / 1e6:.1f}M tentative collisions")
    assert counts.sum() == len(ph) and counts.max() <= tc.max_bounces - 1
    assert np.all(np.isin(ph["g_index"], [0, 1, 2]))
    assert np.all(np.isfinite(ph["power"])) and np.all(ph["power"] >= 0)
    assert np.all((ph["position"] >= -1e-6) & (ph["position"] <= 1 + 1e-6))
    assert np.all(np.abs(np.linalg.norm(ph["direction"].astype(np.float64), axis=1) - 1) < 1e-5)
    pair = np.repeat(np.arange(tc.n_total) % 6, counts)
    bound = LIGHTS2[pair // 3, 3:6] / res.emitted_per_pair[pair][:, None] / tc.rr_max_survival
    assert np.all(ph["power"] <= bound * (1 + 1e-6))
    # phase tags of emitted photons are exactly stratified; deposits roughly so
    h = np.bincount(ph["g_index"], minlength=3)
    assert h.min() > 0.8 * h.max()
    # KNN from the resident trace vs from the fetched copy
    r = np.random.default_rng(0)
    q = r.random((4096, 3)).astype(np.float32)
    g = r.integers(0, 3, 4096).astype(np.uint8)
    ctx.knn_build_traced(res.phase_set)
    i1, d1, c1 = ctx.knn_query(q, g, 32)
    ctx.knn_build(ph, res.phase_set)
    i2, d2, c2 = ctx.knn_query(q, g, 32)
    assert np.array_equal(i1, i2) and np.array_equal(c1, c2)
    kd = oracle.KdTree(ph)
    for k in range(0, 4096, 512):
        ri, rd = kd.knn(q[k], int(g[k]), 32)
        assert np.array_equal(i1[k, :c1[k]], ri)
