"""Render config-2 frames with the comparison renderers (for ncu).  Not part of the product."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2304_07338_b200 import Context, PathTraceConfig, RenderConfig, TraceConfig  # noqa: E402

vol, tf, lights, cam = bench.scene_inputs()
with Context(0) as ctx:
    ctx.upload_volume(vol)
    ctx.set_medium(tf, 100.0)
    ctx.set_lights(lights)
    import torch
    frame = torch.zeros((bench.H_, bench.W_, 3), device="cuda")
    rc = RenderConfig(spp=bench.SPP, seed=bench.SEED, mode="fast")
    for _ in range(2):
        ctx.render_path_traced(cam, rc, PathTraceConfig(), out=frame)
    tc = TraceConfig(n_total=1_000_000, seed=3)
    ctx.trace_photons(tc, device=True)
    ctx.knn_build_traced(tc.phase_set)
    for _ in range(2):
        ctx.render_photon_map(cam, rc, K=64, out=frame)
    torch.cuda.synchronize()
