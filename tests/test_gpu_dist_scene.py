"""Scene replication + sharded KNN targets, world_size 2 on
ONE GPU over gloo: rank 0 broadcasts volume / TF / lights / field / photon map
(dist.broadcast_scene), every rank renders the same frame byte-identically to
a single-process context, and dist.knn_targets_sharded returns the
single-process training targets byte for byte."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
PHASES = [-0.75, 0.0, 0.75]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    from paper_2304_07338_b200 import FieldConfig
    from paper_2304_07338_b200.scene import default_lights, synth_photons, synth_volume, tf_scene_b
    fc = FieldConfig.desk()
    ph = synth_photons(50_000, 3, seed=9)
    r = np.random.default_rng(4)
    n = 3001
    q = (r.random((n, 3)).astype(np.float32), r.normal(size=(n, 3)), r.integers(0, 3, n).astype(np.uint8))
    q[1][:] /= np.linalg.norm(q[1], axis=1, keepdims=True)
    return (synth_volume("sphere_sinusoid", 32), tf_scene_b(), default_lights(), fc,
            fc.init_params(seed=5, embed_scale=0.3, bias_scale=0.1), ph, q)


def _render(ctx):
    from paper_2304_07338_b200 import RenderConfig
    from paper_2304_07338_b200.scene import CameraSpec
    return ctx.render_neural(CameraSpec(80, 60), RenderConfig(spp=2, g=0.0, seed=3, mode="fast"))


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2304_07338_b200 import Context
    from paper_2304_07338_b200.dist import broadcast_scene, knn_targets_sharded
    ctx = Context(0)
    vol, tf, li, fc, par, ph, (x, w, g) = _inputs()
    if rank == 0:
        broadcast_scene(ctx, vol, tf, 100.0, li, (fc, par), ph, PHASES)
    else:
        broadcast_scene(ctx)
    img = _render(ctx)
    t = knn_targets_sharded(ctx, x, w, g, K=32, r_max=0.2)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), img=img, t=t)
    ctx.close()
    dist.destroy_process_group()


def test_scene_broadcast_and_sharded_targets_match_single_gpu(ctx, tmp_path):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    vol, tf, li, fc, par, ph, (x, w, g) = _inputs()
    ctx.upload_volume(vol)
    ctx.set_medium(tf, 100.0)
    ctx.set_lights(li)
    ctx.load_field(fc, par)
    ctx.knn_build(ph, PHASES)
    img = _render(ctx)
    t = ctx.knn_targets(x, w, g, 32, 0.2)
    for r in range(2):
        d = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(d["img"].view(np.uint32), img.view(np.uint32)), r
        assert np.array_equal(d["t"].view(np.uint64), t.view(np.uint64)), r
