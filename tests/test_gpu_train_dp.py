"""Data-parallel field training, world_size 2 on ONE GPU.

Each rank runs pf_train_backward on its half of the step's queries, the
gradient state is all-reduced (gloo here, NCCL on a multi-GPU box) and every
rank applies Adam.  Table gradients are int64 fixed point, so their sum is
exact and order-independent: after one step the hash tables must be
BIT-IDENTICAL to a single-process step over the full batch.  MLP gradients are
binary32 sums in a different order -> MLP updates within 1e-4 of the update
scale (~lr); the loss
(a binary64 sum of two partial sums) relative 1e-12.  Over several steps both
ranks stay bit-identical to each other (same reduced inputs, same Adam).
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
N, STEPS = 4096, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch(n, seed):
    r = np.random.default_rng(seed)
    return (r.random((n, 3)).astype(np.float32), r.random((n, 2)).astype(np.float32),
            r.choice([-0.75, 0.0, 0.75], n).astype(np.float32), r.random((n, 3)).astype(np.float32))


def _setup():
    from paper_2304_07338_b200 import FieldConfig
    fc = FieldConfig.desk()
    return fc, fc.init_params(seed=21, embed_scale=0.1, bias_scale=0.05)


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2304_07338_b200 import Context
    from paper_2304_07338_b200.dist import train_step_dp
    ctx = Context(0)
    fc, params = _setup()
    ctx.train_init(fc, params)
    losses = []
    for s in range(STEPS):
        b = _batch(N, 100 + s)
        lo, hi = rank * N // world, (rank + 1) * N // world
        losses.append(train_step_dp(ctx, *(a[lo:hi] for a in b), n_global=N, step=s, total=STEPS))
        if s == 0:
            np.save(os.path.join(out_dir, f"p1_{rank}.npy"), ctx.train_params())
    np.save(os.path.join(out_dir, f"pN_{rank}.npy"), ctx.train_params())
    np.save(os.path.join(out_dir, f"loss_{rank}.npy"), np.array(losses))
    ctx.close()
    dist.destroy_process_group()


def test_data_parallel_step_matches_full_batch(ctx, oracle, tmp_path):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    fc, params = _setup()
    ctx.train_init(fc, params)
    ref_loss = ctx.train_step(*_batch(N, 100), step=0, total_steps=STEPS)
    ref = ctx.train_params()
    n_tab = len(ref) - oracle._mlp_count(fc)
    p0, p1 = np.load(tmp_path / "p1_0.npy"), np.load(tmp_path / "p1_1.npy")
    assert np.array_equal(p0.view(np.uint32), p1.view(np.uint32))
    assert np.array_equal(p0[:n_tab].view(np.uint32), ref[:n_tab].view(np.uint32)), "table params differ"
    # MLP: a reordered binary32 gradient sum perturbs each update by binary32
    # noise only -- bounded against the step's update scale (~lr)
    du = p0[n_tab:].astype(np.float64) - params[n_tab:]
    dr = ref[n_tab:].astype(np.float64) - params[n_tab:]
    err = np.abs(du - dr).max() / np.abs(dr).max()
    print("mlp update max err / update scale", err, "differing", np.count_nonzero(du != dr), "of", len(du))
    assert err < 1e-4
    l0 = np.load(tmp_path / "loss_0.npy")
    assert abs(l0[0] - ref_loss) <= 1e-12 * ref_loss
    assert np.array_equal(l0, np.load(tmp_path / "loss_1.npy"))
    assert np.array_equal(np.load(tmp_path / "pN_0.npy").view(np.uint32), np.load(tmp_path / "pN_1.npy").view(np.uint32))
