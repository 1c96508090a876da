"""Tile gather over peer memory (pf_ipc_frame_*), world_size 2 on ONE GPU.

Rank 0 allocates the frame and exports its CUDA IPC handle; rank 1 maps it
and renders its interleaved tiles straight into it (the compose kernel's own
stores are the gather -- over NVLink on a multi-GPU box, within the device
here).  Rank 0's frame must be byte-identical to a single-process render,
like the NCCL pack / all_gather / unpack path.  gloo only
carries the 64-byte handle and the barriers.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
W, H = 100, 70


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene(ctx):
    from paper_2304_07338_b200 import FieldConfig
    from paper_2304_07338_b200.scene import default_lights, synth_volume, tf_scene_b
    ctx.upload_volume(synth_volume("sphere_sinusoid", 32))
    ctx.set_medium(tf_scene_b(), 100.0)
    ctx.set_lights(default_lights())
    fc = FieldConfig.desk()
    ctx.load_field(fc, fc.init_params(seed=2, embed_scale=0.3, bias_scale=0.1))


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2304_07338_b200 import Context, RenderConfig
    from paper_2304_07338_b200.scene import CameraSpec
    ctx = Context(0)
    _scene(ctx)
    for mode in ("fast", "parity"):
        obj = [None]
        if rank == 0:
            frame, obj[0] = ctx.ipc_frame_create(H, W)
        dist.broadcast_object_list(obj, src=0)
        if rank != 0:
            frame = ctx.ipc_frame_open(obj[0], H, W)
        rc = RenderConfig(spp=2, g=0.3, seed=7, mode=mode, tile=(16, 16), shard_index=rank, shard_count=world)
        ctx.render_neural(CameraSpec(W, H), rc, out=frame)
        ctx.synchronize()
        dist.barrier()
        if rank == 0:
            np.save(os.path.join(out_dir, f"{mode}.npy"), frame.cpu().numpy())
        dist.barrier()
        if rank != 0:
            frame._pf_holder.release()
        dist.barrier()
        if rank == 0:
            frame._pf_holder.release()
    ctx.close()
    dist.destroy_process_group()


def test_peer_memory_gather_is_byte_identical(ctx, tmp_path):
    from paper_2304_07338_b200 import RenderConfig
    from paper_2304_07338_b200.scene import CameraSpec
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    _scene(ctx)
    for mode in ("fast", "parity"):
        got = np.load(tmp_path / f"{mode}.npy")
        ref = ctx.render_neural(CameraSpec(W, H), RenderConfig(spp=2, g=0.3, seed=7, mode=mode, tile=(16, 16)))
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), mode
