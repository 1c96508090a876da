"""N > 1 tile sharding + gather, world_size 2 over gloo on CPU.

Each rank renders only its interleaved tiles (with the CPU oracle standing in
for the GPU renderer -- tests may use it), the tiles are exchanged with the
product's pack / all_gather / unpack logic, and rank 0's frame must be
byte-identical to a single-process render (frame identical
for any GPU count).
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
W, H, TW, TH = 52, 37, 16, 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _render_tiles(rank, world):
    sys.path.insert(0, str(ROOT))
    from oracle import oracle as o
    from paper_2304_07338_b200 import RenderConfig
    from paper_2304_07338_b200.dist import shard_tiles, tile_rect
    from paper_2304_07338_b200.scene import CameraSpec, default_lights, synth_volume, tf_scene_b
    sc = o.OracleScene(synth_volume("sphere_sinusoid", 24), tf_scene_b(), 100.0)
    rc = RenderConfig(spp=2, g=0.2, seed=5, mode="parity", use_field=False)
    img = np.zeros((H, W, 3), np.float32)
    for t in shard_tiles(W, H, TW, TH, rank, world):
        part, _ = o.render_neural(sc, default_lights(), None, None, CameraSpec(W, H), rc,
                                  rect=tile_rect(t, W, H, TW, TH))
        x0, y0, x1, y1 = tile_rect(t, W, H, TW, TH)
        img[y0:y1, x0:x1] = part[y0:y1, x0:x1]
    return img


def _worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2304_07338_b200.dist import gather_frame_host
    local = torch.from_numpy(_render_tiles(rank, world))
    frame = gather_frame_host(local, W, H, TW, TH)
    if rank == 0:
        np.save(out_path, frame.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_render_gather_is_byte_identical(tmp_path, world):
    out = tmp_path / "frame.npy"
    mp.spawn(_worker, args=(world, _free_port(), str(out)), nprocs=world, join=True)
    got = np.load(out)
    ref = _render_tiles(0, 1)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_tile_cover_properties():
    from paper_2304_07338_b200.dist import _check_cover, packed_floats, shard_tiles
    for count in (1, 2, 3, 4, 8):
        assert _check_cover(1920, 1080, 16, 16, count)
        assert _check_cover(W, H, TW, TH, count)
        sizes = [len(shard_tiles(1920, 1080, 16, 16, s, count)) for s in range(count)]
        assert max(sizes) * 16 * 16 * 3 == packed_floats(1920, 1080, 16, 16, count)


class _ShardCtx:
    """Stands in for Context in train_step_dp on CPU: the oracle computes this
    rank's shard gradient (scaled to its part of the global mean), stored the
    way the device keeps it (int64 2^-40 fixed-point tables, float32 MLP,
    uint8 touched flags)."""

    def __init__(self, fc, params):
        sys.path.insert(0, str(ROOT))
        from oracle import oracle as o
        self.o, self.fc, self.params = o, fc, params
        self.n_tab = len(params) - o._mlp_count(fc)

    def train_backward(self, x, w, g, t, n_global):
        import torch
        loss, grad, touched = self.o.train_grad(self.fc, self.params, x, w, g, t)
        s = len(x) / n_global
        self.gtab = torch.from_numpy(np.rint(grad[:self.n_tab] * s * 2.0 ** 40).astype(np.int64))
        self.gmlp = torch.from_numpy((grad[self.n_tab:] * s).astype(np.float32))
        self.touched = torch.from_numpy(touched.astype(np.uint8))
        return loss * s

    def train_grad_tensors(self):
        return self.gtab, self.gmlp, self.touched

    def synchronize(self):
        pass

    def train_apply(self, step, total):
        self.applied = (step, total)


def _dp_batch():
    r = np.random.default_rng(3)
    n = 48
    return [r.random((n, 3)), r.random((n, 2)), r.choice([-0.75, 0.0, 0.75], n), r.random((n, 3))]


def _dp_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2304_07338_b200 import FieldConfig
    from paper_2304_07338_b200.dist import train_step_dp
    fc = FieldConfig.desk()
    ctx = _ShardCtx(fc, fc.init_params(seed=4, embed_scale=0.1, bias_scale=0.05).astype(np.float64))
    b = _dp_batch()
    n = len(b[0])
    lo, hi = rank * n // world, (rank + 1) * n // world
    loss = train_step_dp(ctx, *(a[lo:hi] for a in b), n_global=n, step=2, total=10)
    assert ctx.applied == (2, 10)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), loss=loss, gtab=ctx.gtab.numpy(), gmlp=ctx.gmlp.numpy(),
             touched=ctx.touched.numpy())
    dist.destroy_process_group()


def test_data_parallel_gradient_reduction(tmp_path):
    """dist.train_step_dp: SUM of the fixed-point table and MLP gradients, MAX
    of the touched flags, SUM of the loss parts == the full-batch step."""
    mp.spawn(_dp_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    sys.path.insert(0, str(ROOT))
    from oracle import oracle as o
    from paper_2304_07338_b200 import FieldConfig
    fc = FieldConfig.desk()
    params = fc.init_params(seed=4, embed_scale=0.1, bias_scale=0.05).astype(np.float64)
    loss, grad, touched = o.train_grad(fc, params, *_dp_batch())
    n_tab = len(params) - o._mlp_count(fc)
    r0, r1 = np.load(tmp_path / "r0.npz"), np.load(tmp_path / "r1.npz")
    for k in ("gtab", "gmlp", "touched", "loss"):
        assert np.array_equal(r0[k], r1[k]), k
    assert abs(float(r0["loss"]) - loss) <= 1e-12 * loss
    assert np.array_equal(r0["touched"], touched.astype(np.uint8))
    assert np.max(np.abs(r0["gtab"] / 2.0 ** 40 - grad[:n_tab])) <= 4e-12
    assert np.allclose(r0["gmlp"], grad[n_tab:], rtol=1e-5, atol=1e-7 * np.abs(grad[n_tab:]).max())


class _RecCtx:
    """Records what broadcast_scene uploads; knn_targets is a per-row function."""

    def __init__(self):
        self.got = {}

    def upload_volume(self, v):
        self.got["volume"] = np.asarray(v).copy()

    def set_medium(self, tf, ds):
        self.got["tf"], self.got["ds"] = np.asarray(tf).copy(), ds

    def set_lights(self, li):
        self.got["lights"] = np.asarray(li).copy()

    def load_field(self, fc, params):
        self.got["fc"], self.got["params"] = fc, np.asarray(params).copy()

    def knn_targets(self, x3, w3, gidx, K, r_max, psi):
        return np.asarray(x3, np.float64) * 2.0 + np.asarray(w3) * K + np.asarray(gidx)[:, None] / psi


def _scene_arrays():
    from paper_2304_07338_b200 import FieldConfig
    from paper_2304_07338_b200.scene import default_lights, synth_volume, tf_scene_b
    fc = FieldConfig.desk()
    return synth_volume("sphere_sinusoid", 12), tf_scene_b(), default_lights(), fc, fc.init_params(seed=3)


def _bq_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2304_07338_b200.dist import broadcast_scene, knn_targets_sharded
    ctx = _RecCtx()
    if rank == 0:
        vol, tf, li, fc, par = _scene_arrays()
        broadcast_scene(ctx, vol, tf, 50.0, li, (fc, par))
    else:
        broadcast_scene(ctx)
    r = np.random.default_rng(1)
    n = 37  # not a multiple of the world size
    x, w, g = r.random((n, 3)).astype(np.float32), r.random((n, 3)), r.integers(0, 3, n).astype(np.uint8)
    t = knn_targets_sharded(ctx, x, w, g, K=8, r_max=0.5, psi=5.0)
    np.savez(os.path.join(out_dir, f"s{rank}.npz"), t=t, ds=ctx.got["ds"],
             **{k: ctx.got[k] for k in ("volume", "tf", "lights", "params")})
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_scene_broadcast_and_sharded_targets(tmp_path, world):
    mp.spawn(_bq_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    vol, tf, li, fc, par = _scene_arrays()
    r = np.random.default_rng(1)
    n = 37
    x, w, g = r.random((n, 3)).astype(np.float32), r.random((n, 3)), r.integers(0, 3, n).astype(np.uint8)
    ref = _RecCtx().knn_targets(x, w, g, 8, 0.5, 5.0)
    for k in range(world):
        d = np.load(tmp_path / f"s{k}.npz")
        assert np.array_equal(d["volume"], vol) and np.array_equal(d["tf"], tf)
        assert np.array_equal(d["lights"], li) and np.array_equal(d["params"], par) and float(d["ds"]) == 50.0
        assert np.array_equal(d["t"], ref)
