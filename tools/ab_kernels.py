"""Times the FP64 photon tracer, the FAST path tracer and the PARITY render
tracer on the config-2 scene (device events) -- for launch-bounds A/B runs."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2304_07338_b200 import Context, FieldConfig, PathTraceConfig, RenderConfig, TraceConfig  # noqa: E402

if __name__ == "__main__":
    import numpy as np
    import torch
    vol, tf, lights, cam = bench.scene_inputs()
    with Context(0) as ctx:
        ctx.upload_volume(vol)
        ctx.set_medium(tf, 100.0)
        ctx.set_lights(lights)
        fc = FieldConfig.paper()
        ctx.load_field(fc, fc.init_params(seed=bench.SEED, embed_scale=1e-2))
        ctx.set_timing(True)
        frame = torch.zeros((bench.H_, bench.W_, 3), device="cuda")
        out = {}
        tc = TraceConfig(n_total=1_000_000, seed=3)
        ts = []
        for _ in range(4):
            ctx.trace_photons(tc, device=True)
            ts.append(ctx.trace_stats()["ms_trace"])
        out["photon_trace_ms"] = float(np.median(ts[1:]))
        rc = RenderConfig(spp=bench.SPP, seed=bench.SEED, mode="fast")
        out["pt_fast_ms"] = float(np.median([ctx.render_path_traced(cam, rc, PathTraceConfig(), out=frame, stats=True)[1]["ms_trace"]
                                             for _ in range(4)][1:]))
        rp = RenderConfig(spp=bench.SPP, seed=bench.SEED, mode="parity")
        out["parity_trace_ms"] = float(np.median([ctx.render_neural(cam, rp, out=frame, stats=True)[1]["ms_trace"]
                                                  for _ in range(4)][1:]))
        print(json.dumps(out))
