import os, sys, json
sys.path.insert(0, "."); sys.path.insert(0, "tools")
import torch, numpy as np
import bench
from paper_2304_07338_b200 import Context, RenderConfig, TraceConfig
vol, tf, lights, cam = bench.scene_inputs()
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
with Context(0, stream=s.cuda_stream) as ctx:
    ctx.upload_volume(vol); ctx.set_medium(tf, 100.0); ctx.set_lights(lights)
    tc = TraceConfig(n_total=1_000_000, seed=3); ctx.trace_photons(tc, device=True); ctx.knn_build_traced(tc.phase_set)
    frame = torch.zeros((bench.H_, bench.W_, 3), device="cuda")
    rc = RenderConfig(spp=8, seed=bench.SEED, mode="fast")
    for mode in ("0", "1", "0", "1"):
        os.environ["PF_KNN_MERGE"] = mode
        ctx.render_photon_map(cam, rc, K=64, out=frame); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3): ctx.render_photon_map(cam, rc, K=64, out=frame)
        b.record(); torch.cuda.synchronize()
        print("merge" if mode == "1" else "sel", a.elapsed_time(b) / 3, flush=True)
