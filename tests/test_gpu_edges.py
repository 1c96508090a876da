"""Edge cases through the C ABI: empty batches, degenerate photon maps,
device-resident I/O, and the reference's error behaviour."""
import numpy as np
import pytest

from paper_2304_07338_b200 import FieldConfig, RenderConfig
from paper_2304_07338_b200.scene import CameraSpec, default_lights, make_photons, synth_photons, synth_volume, tf_scene_b

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scene(ctx):
    ctx.upload_volume(synth_volume("sphere_sinusoid", 32))
    ctx.set_medium(tf_scene_b(), 100.0)
    ctx.set_lights(default_lights())
    return ctx


def test_empty_batches(scene, oracle):
    ctx = scene
    z3, z1 = np.zeros((0, 3)), np.zeros(0)
    hit, pos, _ = ctx.delta_track_batch(z3, z3, z1, z1, 0, "camera", np.zeros(0, np.uint64))
    assert hit.shape == (0,) and pos.shape == (0, 3)
    assert ctx.transmittance_batch(z3, z3, 0, "nee", np.zeros(0, np.uint64)).shape == (0,)
    assert ctx.rng_doubles(0, "test", np.zeros(0, np.uint64), 3).shape == (0, 3)
    fc = FieldConfig.desk()
    ctx.load_field(fc, fc.init_params(seed=1))
    assert ctx.field_query(np.zeros((0, 3), np.float32), np.zeros((0, 2), np.float32),
                           np.zeros(0, np.float32)).shape == (0, 3)
    ctx.knn_build(synth_photons(100, 3, seed=1), [-0.75, 0.0, 0.75])
    ids, d2, cnt = ctx.knn_query(np.zeros((0, 3), np.float32), np.zeros(0, np.uint8), 8)
    assert ids.shape == (0, 8) and cnt.shape == (0,)


def test_knn_k_exceeds_population_and_bad_tags(scene, oracle):
    ctx = scene
    ph = synth_photons(300, 3, seed=2)
    ph["g_index"][:50] = 7                      # tags outside the phase set are never returned
    ctx.knn_build(ph, [-0.75, 0.0, 0.75])
    r = np.random.default_rng(3)
    q = r.random((64, 3)).astype(np.float32)
    g = r.integers(0, 3, 64).astype(np.uint8)
    ids, d2, cnt = ctx.knn_query(q, g, 1024)     # K > photons of any phase
    for i in range(64):
        ri, rd = oracle.knn_brute(ph, q[i], int(g[i]), 1024)
        assert cnt[i] == len(ri) and np.array_equal(ids[i, :cnt[i]], ri)
    ids, _, cnt = ctx.knn_query(q, np.full(64, 5, np.uint8), 8)  # unknown phase -> empty
    assert np.all(cnt == 0) and np.all(ids == 0xFFFFFFFF)
    _, _, cnt = ctx.knn_query(q, g, 8, 1e-6)      # tiny radius
    assert np.all(cnt == 0)
    with pytest.raises(ValueError):
        ctx.knn_query(q, g, 0)
    with pytest.raises(ValueError):
        ctx.knn_query(q, g, 8, 0.0)


def test_knn_coincident_photons(scene, oracle):
    """All photons at one point: d2 ties everywhere -> order by id; Eq. 6 r < 1e-6 guard."""
    ctx = scene
    n = 500
    ph = make_photons(np.full((n, 3), 0.25, np.float32), np.tile([0, 0, 1], (n, 1)).astype(np.float32),
                      np.ones((n, 3), np.float32), np.zeros(n))
    ctx.knn_build(ph, [0.0])
    ids, d2, cnt = ctx.knn_query(np.array([[0.25, 0.25, 0.25], [0.9, 0.9, 0.9]], np.float32),
                                 np.zeros(2, np.uint8), 64)
    assert list(ids[0]) == list(range(64)) and np.all(d2[0] == 0.0)
    assert list(ids[1]) == list(range(64))
    tg = ctx.knn_targets(np.array([[0.25, 0.25, 0.25]], np.float32), np.array([[0, 0, 1.0]]),
                         np.zeros(1, np.uint8), 64)
    assert np.all(tg == 1.0)                      # r = 0 -> L = 0 -> encode_log(0) = 1


def test_device_resident_io_matches_host(scene):
    import torch
    ctx = scene
    cam = CameraSpec(64, 48)
    rc = RenderConfig(spp=2, seed=3, mode="fast", use_field=False)
    host = ctx.render_neural(cam, rc)
    dev = torch.zeros((48, 64, 3), device="cuda")
    ctx.render_neural(cam, rc, out=dev)
    ctx.synchronize()
    assert np.array_equal(dev.cpu().numpy(), host)
    r = np.random.default_rng(0)
    o = r.uniform(0, 1, (512, 3))
    d = r.standard_normal((512, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    idx = np.arange(512, dtype=np.uint64)
    t = ctx.transmittance_batch(o, o + d, 1, "nee", idx, 2)
    td = ctx.transmittance_batch(torch.tensor(o, device="cuda"), torch.tensor(o + d, device="cuda"), 1, "nee",
                                 torch.tensor(idx.astype(np.int64), device="cuda"), 2)
    assert np.array_equal(t, td)


def test_render_background_only_outside_volume(scene):
    """Camera looking away from the volume: every sample misses -> background."""
    img, st = scene.render_neural(CameraSpec(32, 32, (0.5, 0.5, -0.9), (0.5, 0.5, -2.0), (0, 1, 0), 30.0),
                                  RenderConfig(spp=4, background=(0.25, 0.5, 0.75), use_field=False), stats=True)
    assert st["hits"] == 0 and np.all(img == np.array([0.25, 0.5, 0.75], np.float32))


def test_async_host_frames_equal_sync(ctx):
    """pf_render_neural_async: pipelined host frames equal the synchronous API's."""
    import torch
    from paper_2304_07338_b200 import FieldConfig, RenderConfig
    from paper_2304_07338_b200.scene import CameraSpec, default_lights, synth_volume, tf_scene_b
    ctx.upload_volume(synth_volume("sphere_sinusoid", 32))
    ctx.set_medium(tf_scene_b(), 100.0)
    ctx.set_lights(default_lights())
    fc = FieldConfig.desk()
    ctx.load_field(fc, fc.init_params(seed=3, embed_scale=0.3, bias_scale=0.1))
    cam = CameraSpec(64, 40)
    cfgs = [RenderConfig(spp=2, seed=s, mode=m) for s, m in [(1, "fast"), (2, "parity"), (3, "fast"), (4, "fast")]]
    want = [ctx.render_neural(cam, c) for c in cfgs]
    bufs = [torch.zeros((40, 64, 3), dtype=torch.float32).pin_memory() for _ in range(2)]
    got = []
    for i, c in enumerate(cfgs):
        ctx.render_neural_async(cam, c, bufs[i % 2].numpy())
        if i > 0:
            ctx.frame_wait(bufs[(i - 1) % 2].numpy())
            got.append(bufs[(i - 1) % 2].numpy().copy())
    ctx.frame_wait(bufs[(len(cfgs) - 1) % 2].numpy())
    got.append(bufs[(len(cfgs) - 1) % 2].numpy().copy())
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
    with pytest.raises(ValueError):
        ctx.frame_wait(np.zeros((40, 64, 3), np.float32))


def test_async_frames_with_shards_and_errors(ctx):
    """Async host frames of a shard (other tiles zero) and the API's error paths
    for the IPC frame and the optimizer state."""
    import torch
    from paper_2304_07338_b200 import FieldConfig, RenderConfig
    from paper_2304_07338_b200 import _lib
    from paper_2304_07338_b200.scene import CameraSpec, default_lights, synth_volume, tf_scene_b
    ctx.upload_volume(synth_volume("sphere_sinusoid", 24))
    ctx.set_medium(tf_scene_b(), 100.0)
    ctx.set_lights(default_lights())
    fc = FieldConfig.desk()
    ctx.load_field(fc, fc.init_params(seed=1, embed_scale=0.2))
    cam = CameraSpec(48, 32)
    rc = RenderConfig(spp=2, seed=5, mode="fast", tile=(16, 16), shard_index=1, shard_count=2)
    buf = torch.full((32, 48, 3), 7.0, dtype=torch.float32).pin_memory()
    ctx.render_neural_async(cam, rc, buf.numpy())
    ctx.frame_wait(buf.numpy())
    dev = torch.zeros((32, 48, 3), dtype=torch.float32, device="cuda")
    ctx.render_neural(cam, rc, out=dev)
    ctx.synchronize()
    assert np.array_equal(buf.numpy(), dev.cpu().numpy())   # untouched shards are zero, not stale
    # IPC handle of nothing -> runtime error (never a silent fallback)
    with pytest.raises(RuntimeError):
        ctx.ipc_frame_open(bytes(64), 32, 48)
    # optimizer state of the wrong size -> invalid argument
    ctx.train_init(fc, fc.init_params(seed=1))
    n, _ = ctx.train_counts()
    bad = np.zeros(n - 1, np.float32)
    rc_ = _lib.lib().pf_train_state_set(ctx._h, bad.ctypes.data, bad.ctypes.data, bad.ctypes.data, n - 1)
    assert rc_ == 1
