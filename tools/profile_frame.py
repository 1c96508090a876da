"""Render config-2 frames (for ncu / launch lists).  Not part of the product."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2304_07338_b200 import Context, FieldConfig, RenderConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="fast")
ap.add_argument("--frames", type=int, default=3)
ap.add_argument("--field", default="paper")
a = ap.parse_args()
vol, tf, lights, cam = bench.scene_inputs()
with Context(0) as ctx:
    ctx.upload_volume(vol)
    ctx.set_medium(tf, 100.0)
    ctx.set_lights(lights)
    fc = getattr(FieldConfig, a.field)()
    ctx.load_field(fc, fc.init_params(seed=bench.SEED, embed_scale=1e-2))
    import torch
    frame = torch.zeros((bench.H_, bench.W_, 3), device="cuda")
    rc = RenderConfig(spp=bench.SPP, seed=bench.SEED, mode=a.mode)
    for i in range(a.frames):
        _, st = ctx.render_neural(cam, rc, out=frame, stats=True)
    print(st)
