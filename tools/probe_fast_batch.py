"""Probe: FAST-mode delta_track_batch hit count on the tracking-test rays, optionally after
holding <GB> of device memory first (allocation placement).  Tooling for the DDA bounds bug."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2304_07338_b200 import Context
from paper_2304_07338_b200.scene import synth_volume, tf_scene_a
gb = float(sys.argv[1])
hold = torch.empty(int(gb * 2**30), dtype=torch.uint8, device="cuda") if gb > 0 else None
ctx = Context(0)
ctx.upload_volume(synth_volume("sphere_sinusoid", 64))
ctx.set_medium(tf_scene_a(), 100.0)
n = 200000
r = np.random.default_rng(8)
o = np.tile([0.5, 0.5, -0.9], (n, 1))
d = np.column_stack([r.uniform(-0.3, 0.3, n), r.uniform(-0.3, 0.3, n), np.ones(n)])
d /= np.linalg.norm(d, axis=1, keepdims=True)
idx = np.arange(n, dtype=np.uint64)
h, p, _ = ctx.delta_track_batch(o, d, np.zeros(n), np.full(n, np.inf), 5, "camera", idx, fp64=False)
print("ok", gb, h.sum())
hp, pp, _ = ctx.delta_track_batch(o, d, np.zeros(n), np.full(n, np.inf), 5, "camera", idx, fp64=True)
print("parity hits", hp.sum())
