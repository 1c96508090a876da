"""Hashes of every kernel family's output on fixed inputs, optionally after
holding <GiB> of device memory first: a kernel whose results change with the
allocation placement reads memory it does not own (how the FAST batch DDA
miscompile showed up).  Tooling, not product.

usage: python tools/placement_check.py [GiB]
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2304_07338_b200 import Context, FieldConfig, RenderConfig  # noqa: E402
from paper_2304_07338_b200.api import TraceConfig  # noqa: E402


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:12]


if __name__ == "__main__":
    import torch
    gib = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
    hold = torch.empty(int(gib * 2**30), dtype=torch.uint8, device="cuda") if gib > 0 else None
    vol, tf, lights, cam = bench.scene_inputs()
    out = {}
    with Context(0) as ctx:
        ctx.upload_volume(vol)
        ctx.set_medium(tf, 100.0)
        ctx.set_lights(lights)
        fc = FieldConfig.paper()
        ctx.load_field(fc, fc.init_params(seed=bench.SEED, embed_scale=1e-2))
        for mode in ("parity", "fast"):
            rc = RenderConfig(spp=4, seed=bench.SEED, mode=mode)
            out[f"neural_{mode}"] = h(ctx.render_neural(cam, rc))
            out[f"path_{mode}"] = h(ctx.render_path_traced(cam, rc))
        tc = TraceConfig(n_total=200_000, seed=3)
        tr = ctx.trace_photons(tc)
        out["photons"] = h(tr.photons)
        ctx.knn_build(tr.photons, tc.phase_set)
        x, w, g, t = ctx.make_batch(11, 0, 1 << 14, 64)
        out["knn_targets"] = h(t)
        r = np.random.default_rng(1)
        q = ctx.field_query(r.random((1 << 14, 3), dtype=np.float32), r.random((1 << 14, 2), dtype=np.float32),
                            np.zeros(1 << 14, np.float32))
        out["field_query"] = h(q)
        n = 100_000
        o = np.tile([0.5, 0.5, -0.9], (n, 1))
        d = np.column_stack([r.uniform(-0.3, 0.3, n), r.uniform(-0.3, 0.3, n), np.ones(n)])
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        idx = np.arange(n, dtype=np.uint64)
        for fp64 in (True, False):
            hit, pos, _ = ctx.delta_track_batch(o, d, np.zeros(n), np.full(n, np.inf), 5, "camera", idx, fp64=fp64)
            out[f"batch_{'parity' if fp64 else 'fast'}"] = h(hit) + "/" + h(pos[hit == 1])
        b = np.tile([2.0, 2.5, -1.0], (n, 1))
        out["transmittance_ratio"] = h(ctx.transmittance_batch(o + 0.9 * d, b, 21, "nee", idx, 2, ratio=True))
    print(gib, " ".join(f"{k}={v}" for k, v in out.items()))
