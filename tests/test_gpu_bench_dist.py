"""bench.py itself at N = 2 (torchrun, one process per rank) on ONE GPU:
PF_BENCH_ONE_DEVICE=1 puts both ranks on cuda:0 and the collectives on gloo
(NCCL refuses two ranks on one device).  For both tile gathers -- "p2p" (each
rank's compose kernel stores its tiles into rank 0's frame through a CUDA IPC
mapping) and "nccl" (pack / all-gather / unpack) -- rank 0's headline frame
must be byte-identical to the N = 1 frame (the SPEC.md:734
worker-count invariance applied to the bench path), and the bench line must
carry the per-N roofline and e2e fields.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
ARGS = ["--steps", "2", "--warmup", "3", "--no-extras", "--no-cpu-baseline", "--no-fast"]


def _run(tmp_path, n, gather, port):
    dump = tmp_path / f"frame_{n}_{gather}.npy"
    env = dict(os.environ, PF_BENCH_DUMP=str(dump), PYTHONPATH=str(ROOT))
    if n == 1:
        cmd = [sys.executable, str(ROOT / "bench.py"), *ARGS]
    else:
        env.update(PF_BENCH_ONE_DEVICE="1", PF_DIST_BACKEND="gloo", PF_GATHER=gather)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
               "--gpus", str(n), *ARGS]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return np.load(dump), lines[0]


def test_bench_n2_frames_match_n1(tmp_path):
    f1, l1 = _run(tmp_path, 1, "none", 0)
    assert l1["n_gpus"] == 1 and l1["dtype"] == "f64"
    for i, gather in enumerate(["p2p", "nccl"]):
        f2, l2 = _run(tmp_path, 2, gather, 29511 + i)
        print(gather, l2["value"], l2["config"]["gather"], l2["roofline"]["frac"], l2["e2e"]["value"])
        assert l2["n_gpus"] == 2 and l2["config"]["gather"] == gather
        assert l2["roofline"]["achieved"] > 0 and l2["e2e"]["value"] > 0
        assert np.array_equal(f1.view(np.uint32), f2.view(np.uint32)), gather
