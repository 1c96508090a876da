"""Reference-produced golden vectors (tests/golden/reference_c1.npz, generated
by tests/golden/make_golden.py from the UNMODIFIED reference via oracle/_ref).

CPU: the C restatement must reproduce them bit-for-bit.
GPU: the parity kernels must reproduce them (hit decisions / transmittance
outcomes exactly; binary64 positions bitwise except CUDA-vs-glibc log() last-bit
cases, <= 1e-3 of hits and <= 1e-12 absolute).
"""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

from paper_2304_07338_b200 import RenderConfig
from paper_2304_07338_b200.scene import CameraSpec, default_lights

G = np.load(Path(__file__).with_name("golden") / "reference_c1.npz")
CAM, NEE = 3, 4


def test_golden_rng_oracle(oracle):
    for a, sd in enumerate(G["rng_seeds"]):
        for b, st in enumerate(G["rng_streams"]):
            out = np.zeros((len(G["rng_idx"]), 8))
            idx = np.ascontiguousarray(G["rng_idx"])
            oracle.lib().or_rng_doubles(int(sd), int(st), len(idx), idx.ctypes.data, 8, out.ctypes.data)
            assert np.array_equal(out.view(np.uint64), G["rng"][a, b].view(np.uint64))


def _oscene(oracle):
    return oracle.OracleScene(G["vol"], G["tf"], float(G["density"]))


def test_golden_tracking_oracle(oracle):
    sc = _oscene(oracle)
    assert sc.sigma_max == float(G["sigma_max"])
    hit, pos, rgba = sc.delta_track(G["dt_o"], G["dt_d"], G["dt_tmin"], G["dt_tmax"], int(G["dt_seed"]), CAM,
                                    G["dt_idx"])
    assert np.array_equal(hit, G["dt_hit"])
    assert np.array_equal(pos.view(np.uint64), G["dt_pos"].view(np.uint64))
    assert np.array_equal(rgba.view(np.uint64), G["dt_rgba"].view(np.uint64))
    for k, n in (("tr_T1", 1), ("tr_T3", 3)):
        t = sc.transmittance(G["tr_a"], G["tr_b"], int(G["tr_seed"]), NEE, G["tr_idx"], n)
        assert np.array_equal(t, G[k])


def test_golden_render_oracle(oracle):
    sc = _oscene(oracle)
    rc = RenderConfig(spp=int(G["img_spp"]), g=float(G["img_g"]), seed=int(G["img_seed"]), mode="parity",
                      use_field=False, background=(0.05, 0.1, 0.2))
    img, st = oracle.render_neural(sc, default_lights(), None, None, CameraSpec(48, 40), rc)
    assert st["hits"] == int(G["img_hits"])
    assert np.array_equal(img.view(np.uint32), G["img"].view(np.uint32))


@pytest.fixture(scope="module")
def gscene(ctx):
    ctx.upload_volume(G["vol"])
    ctx.set_medium(G["tf"], float(G["density"]))
    ctx.set_lights(default_lights())
    return ctx


@pytest.mark.gpu
def test_golden_rng_gpu(ctx):
    for a, sd in enumerate(G["rng_seeds"]):
        for b, st in enumerate(G["rng_streams"]):
            out = ctx.rng_doubles(int(sd), int(st), G["rng_idx"], 8)
            assert np.array_equal(out.view(np.uint64), G["rng"][a, b].view(np.uint64))


@pytest.mark.gpu
def test_golden_tracking_gpu(gscene):
    ctx = gscene
    assert ctx.sigma_max == float(G["sigma_max"])
    hit, pos, rgba = ctx.delta_track_batch(G["dt_o"], G["dt_d"], G["dt_tmin"], G["dt_tmax"], int(G["dt_seed"]),
                                           CAM, G["dt_idx"], fp64=True)
    assert np.array_equal(hit, G["dt_hit"])
    h = hit == 1
    same = np.all(pos[h].view(np.uint64) == G["dt_pos"][h].view(np.uint64), axis=1)
    assert np.count_nonzero(~same) <= max(2, 1e-3 * h.sum())
    assert np.max(np.abs(pos[h] - G["dt_pos"][h])) < 1e-12
    for k, n in (("tr_T1", 1), ("tr_T3", 3)):
        t = ctx.transmittance_batch(G["tr_a"], G["tr_b"], int(G["tr_seed"]), NEE, G["tr_idx"], n)
        assert np.count_nonzero(t != G[k]) <= 2


@pytest.mark.gpu
def test_golden_render_gpu(gscene):
    rc = RenderConfig(spp=int(G["img_spp"]), g=float(G["img_g"]), seed=int(G["img_seed"]), mode="parity",
                      use_field=False, background=(0.05, 0.1, 0.2))
    img, st = gscene.render_neural(CameraSpec(48, 40), rc, stats=True)
    assert st["hits"] == int(G["img_hits"])
    n_diff = np.count_nonzero(np.any(img != G["img"], axis=2))
    assert n_diff <= 2
    assert np.allclose(img, G["img"], rtol=1e-6, atol=1e-9)
