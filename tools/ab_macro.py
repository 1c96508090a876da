"""A/B of the FAST tracer's macro-cell size (PF_MACRO_CELL, read at context creation)."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2304_07338_b200 import Context, FieldConfig, RenderConfig  # noqa: E402

if __name__ == "__main__":
    import numpy as np
    import torch
    vol, tf, lights, cam = bench.scene_inputs()
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    for v in sys.argv[1].split(","):
        os.environ["PF_MACRO_CELL"] = v
        with Context(0, stream=s.cuda_stream) as ctx:
            ctx.upload_volume(vol)
            ctx.set_medium(tf, 100.0)
            ctx.set_lights(lights)
            fc = FieldConfig.paper()
            ctx.load_field(fc, fc.init_params(seed=bench.SEED, embed_scale=1e-2))
            ctx.set_timing(True)
            frame = torch.zeros((bench.H_, bench.W_, 3), device="cuda")
            rc = RenderConfig(spp=bench.SPP, seed=bench.SEED, mode="fast")
            sts = [ctx.render_neural(cam, rc, out=frame, stats=True)[1] for _ in range(8)][3:]
            print("macro", v, json.dumps({"ms_trace": float(np.mean([x["ms_trace"] for x in sts])),
                                          "steps_per_sample": (sts[-1]["primary_steps"] + sts[-1]["shadow_steps"]) / sts[-1]["samples"],
                                          "hits": sts[-1]["hits"]}), flush=True)
