"""Multi-GPU image-tile sharding.

One process per GPU.  Screen tiles (tile_w x tile_h) are numbered row-major
and interleaved round-robin over the ranks (tile t -> rank t % world), so
screen-space load imbalance averages out and every rank's tile list is static.
Every camera sample owns the RNG stream make_rng(seed, stream, global sample
index), hence the frame is byte-identical for any world size.  Per frame:
  1. each rank renders only its tiles (pf_render_neural with shard_index /
     shard_count) into a local frame buffer;
  2. it packs its tiles contiguously (pf_tiles_pack) into a buffer padded to
     the largest shard's tile count;
  3. one all_gather_into_tensor (NCCL over NVLink/NVSwitch) moves the packed
     tiles; rank 0 de-tiles them into the final frame (pf_tiles_unpack).
The default device path (bench.py, render_frame_p2p) fuses the gather into
the render instead: rank 0 exports its frame buffer (pf_ipc_frame_create,
CUDA IPC), every other rank maps it (pf_ipc_frame_open) and renders with the
mapped pointer as its output, so each rank's compose kernel stores its tiles
straight into rank 0's frame over NVLink peer memory -- no pack, no
collective payload, no unpack; a stream-ordered 1-element all-reduce before
and after the render orders the frames.
The functions below are the host-side statement of that tile map -- the CUDA
kernels implement the same arithmetic -- and a CPU/gloo implementation of the
exchange used to test the N > 1 logic without GPUs.
"""
from __future__ import annotations

import numpy as np


def tile_grid(width: int, height: int, tile_w: int, tile_h: int) -> tuple[int, int]:
    return (width + tile_w - 1) // tile_w, (height + tile_h - 1) // tile_h


def shard_tiles(width, height, tile_w, tile_h, shard, count) -> list[int]:
    tx, ty = tile_grid(width, height, tile_w, tile_h)
    return list(range(shard, tx * ty, count))


def tile_rect(t, width, height, tile_w, tile_h) -> tuple[int, int, int, int]:
    tx, _ = tile_grid(width, height, tile_w, tile_h)
    x0, y0 = (t % tx) * tile_w, (t // tx) * tile_h
    return x0, y0, min(x0 + tile_w, width), min(y0 + tile_h, height)


def packed_floats(width, height, tile_w, tile_h, count) -> int:
    """Per-shard packed buffer length (padded to the largest shard)."""
    tx, ty = tile_grid(width, height, tile_w, tile_h)
    return ((tx * ty + count - 1) // count) * tile_w * tile_h * 3


def pack_tiles(frame, width, height, tile_w, tile_h, shard, count, out=None):
    """Host statement of pf_tiles_pack: tile-major, row-major inside a tile, zero padding."""
    import torch
    per = packed_floats(width, height, tile_w, tile_h, count)
    out = torch.zeros(per, dtype=torch.float32) if out is None else out
    view = out.view(-1, tile_h, tile_w, 3)
    for j, t in enumerate(shard_tiles(width, height, tile_w, tile_h, shard, count)):
        x0, y0, x1, y1 = tile_rect(t, width, height, tile_w, tile_h)
        view[j, : y1 - y0, : x1 - x0] = frame[y0:y1, x0:x1]
    return out


def unpack_tiles(packed_all, width, height, tile_w, tile_h, count, frame):
    """Host statement of pf_tiles_unpack."""
    per = packed_floats(width, height, tile_w, tile_h, count)
    for r in range(count):
        view = packed_all[r * per:(r + 1) * per].view(-1, tile_h, tile_w, 3)
        for j, t in enumerate(shard_tiles(width, height, tile_w, tile_h, r, count)):
            x0, y0, x1, y1 = tile_rect(t, width, height, tile_w, tile_h)
            frame[y0:y1, x0:x1] = view[j, : y1 - y0, : x1 - x0]
    return frame


def gather_frame_host(local_frame, width, height, tile_w, tile_h, group=None):
    """The N > 1 exchange on host tensors (gloo): pack -> all_gather -> unpack on rank 0."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    packed = pack_tiles(local_frame, width, height, tile_w, tile_h, rank, world)
    gathered = torch.empty(packed.numel() * world, dtype=torch.float32)
    dist.all_gather_into_tensor(gathered, packed, group=group)
    if rank != 0:
        return None
    frame = torch.zeros((height, width, 3), dtype=torch.float32)
    return unpack_tiles(gathered, width, height, tile_w, tile_h, world, frame)


def render_frame_sharded(ctx, cam, rc, frame, packed, gathered, group=None):
    """Device path used by bench.py: render own tiles, NCCL all_gather, rank-0 de-tile."""
    import torch.distributed as dist
    ctx.render_neural(cam, rc, out=frame)
    if rc.shard_count == 1:
        return frame
    ctx.tiles_pack(cam, rc, frame, packed)
    dist.all_gather_into_tensor(gathered, packed, group=group)
    if rc.shard_index == 0:
        ctx.tiles_unpack(cam, rc, gathered, packed.numel(), frame)
    return frame


def open_shared_frame(ctx, height, width, group=None):
    """Rank 0 allocates + exports the frame, the other ranks map it (CUDA IPC)."""
    import torch.distributed as dist
    obj = [None]
    frame = None
    if dist.get_rank(group) == 0:
        frame, obj[0] = ctx.ipc_frame_create(height, width)
    dist.broadcast_object_list(obj, src=0, group=group)
    if frame is None:
        frame = ctx.ipc_frame_open(obj[0], height, width)
    return frame


def render_frame_p2p(ctx, cam, rc, shared_frame, sync, group=None):
    """Fused gather: this rank's compose kernel writes its tiles into rank 0's
    frame (peer memory); the all-reduces order it against the previous frame's
    readers and make the frame complete on rank 0."""
    import torch.distributed as dist
    dist.all_reduce(sync, group=group)
    ctx.render_neural(cam, rc, out=shared_frame)
    dist.all_reduce(sync, group=group)
    return shared_frame


def train_step_dp(ctx, x3, wsph2, g, targets3, n_global: int, step: int, total: int, group=None) -> float:
    """Data-parallel train_step (one process per GPU): this rank's shard
    backward, all-reduce of the gradient state (int64 fixed-point table sums --
    exact and order-independent -- float32 MLP sums, touched flags by MAX),
    then Adam on every rank with identical inputs.  Returns the global loss."""
    import torch
    import torch.distributed as dist
    loss = ctx.train_backward(x3, wsph2, g, targets3, n_global)
    gtab, gmlp, touched = ctx.train_grad_tensors()
    ctx.synchronize()
    host = dist.get_backend(group) != "nccl"  # gloo: reduce host copies
    for buf, op in ((gtab, dist.ReduceOp.SUM), (gmlp, dist.ReduceOp.SUM), (touched, dist.ReduceOp.MAX)):
        t = buf.to(torch.int32) if buf.dtype == torch.uint8 else buf
        if host:
            t = t.cpu()
        dist.all_reduce(t, op=op, group=group)
        buf.copy_(t.to(buf.dtype))
    # NCCL reduces device tensors only; gloo host tensors
    lt = torch.tensor([loss], dtype=torch.float64, device="cpu" if host else gtab.device)
    dist.all_reduce(lt, op=dist.ReduceOp.SUM, group=group)
    if gtab.is_cuda:
        torch.cuda.synchronize()
    ctx.train_apply(step, total)
    return float(lt.item())


def _bcast_array(a, src, group, device):
    """Broadcast a numpy array from rank src (shape/dtype travel as an object);
    returns a torch tensor on `device` on every rank."""
    import torch
    import torch.distributed as dist
    meta = [None if a is None else (tuple(a.shape), str(a.dtype))]
    dist.broadcast_object_list(meta, src=src, group=group)
    if meta[0] is None:
        return None
    shape, dt = meta[0]
    if dist.get_rank(group) == src:
        t = torch.from_numpy(np.ascontiguousarray(a)).to(device)
    else:
        t = torch.empty(shape, dtype=getattr(torch, np.dtype(dt).name), device=device)
    dist.broadcast(t, src=src, group=group)
    return t


def broadcast_scene(ctx, volume=None, tf_points=None, density_scale: float = 100.0, lights=None,
                    field=None, photons=None, phase_set=None, src: int = 0, group=None) -> None:
    """Replicate the scene on every rank (volume, TF, lights
    and field weights are broadcast from rank `src` on a scene / TF change and
    uploaded into each rank's context; the photon map likewise, rebuilt into
    each rank's KNN index).  Arguments are only read on `src`; `field` is
    (FieldConfig, params), `photons` a PHOTON_DTYPE array with its phase set.  Large arrays travel as device tensors
    over NCCL (host tensors over gloo); the small TF / light / config records
    as pickled objects."""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    small = [None]
    if dist.get_rank(group) == src:
        small[0] = (None if tf_points is None else np.asarray(tf_points, np.float64), float(density_scale),
                    None if lights is None else np.asarray(lights, np.float64),
                    None if field is None else field[0], None if phase_set is None else list(phase_set))
    dist.broadcast_object_list(small, src=src, group=group)
    tf, ds, li, fc, ps = small[0]
    vol = _bcast_array(None if volume is None else np.asarray(volume, np.float32), src, group, dev)
    par = _bcast_array(None if field is None else np.asarray(field[1], np.float32), src, group, dev)
    phb = _bcast_array(None if photons is None else np.ascontiguousarray(photons).view(np.uint8), src, group, dev)
    if vol is not None:
        ctx.upload_volume(vol)
    if tf is not None:
        ctx.set_medium(tf, ds)
    if li is not None:
        ctx.set_lights(li)
    if fc is not None:
        ctx.load_field(fc, par)
    if phb is not None:
        from .scene import PHOTON_DTYPE
        ctx.knn_build(phb.cpu().numpy().view(PHOTON_DTYPE), ps)
    if dev == "cuda":
        torch.cuda.synchronize()


def shard_rows(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced row range [lo, hi) of rank `rank`."""
    return rank * n // world, (rank + 1) * n // world


def knn_targets_sharded(ctx, x3, w3, gidx, K: int, r_max: float = float("inf"), psi: float = 5.0,
                        group=None) -> np.ndarray:
    """Training targets of a query batch split over ranks (SURVEY.md 8(e),
    KNN C3): each rank runs the KNN gather + Eq. 6/7 on its contiguous share
    of the queries against its replica of the photon map, then one all_gather
    assembles the (n, 3) binary64 targets on every rank.  Queries are
    independent, so the result is byte-identical to a single-GPU call."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    n = int(np.asarray(x3).shape[0])
    lo, hi = shard_rows(n, rank, world)
    part = ctx.knn_targets(np.asarray(x3)[lo:hi], np.asarray(w3)[lo:hi], np.asarray(gidx)[lo:hi], K, r_max, psi)
    per = -(-n // world)  # padded share
    buf = np.zeros((per, 3), np.float64)
    buf[:hi - lo] = part
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.from_numpy(buf).to(dev)
    out = torch.empty((world * per, 3), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(out, t, group=group)
    out = out.cpu().numpy()
    return np.concatenate([out[r * per:r * per + (shard_rows(n, r, world)[1] - shard_rows(n, r, world)[0])]
                           for r in range(world)])


def _check_cover(width, height, tile_w, tile_h, count) -> bool:
    seen = np.zeros((height, width), np.int32)
    for s in range(count):
        for t in shard_tiles(width, height, tile_w, tile_h, s, count):
            x0, y0, x1, y1 = tile_rect(t, width, height, tile_w, tile_h)
            seen[y0:y1, x0:x1] += 1
    return bool(np.all(seen == 1))
