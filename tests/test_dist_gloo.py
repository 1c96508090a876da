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
