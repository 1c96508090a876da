"""A/B of field-path knobs (argv[2], default PF_MLP_WG; e.g. PF_FIELD_FUSED): frame field time +
field microbench + output equality."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2304_07338_b200 import Context, FieldConfig, RenderConfig  # noqa: E402

VAR = sys.argv[2] if len(sys.argv) > 2 else "PF_MLP_WG"

if __name__ == "__main__":
    import numpy as np
    import torch
    vol, tf, lights, cam = bench.scene_inputs()
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    with Context(0, stream=s.cuda_stream) as ctx:
        ctx.upload_volume(vol)
        ctx.set_medium(tf, 100.0)
        ctx.set_lights(lights)
        fc = FieldConfig.paper()
        prm = fc.init_params(seed=bench.SEED, embed_scale=1e-2)
        ctx.set_timing(True)
        frame = torch.zeros((bench.H_, bench.W_, 3), device="cuda")
        rc = RenderConfig(spp=bench.SPP, seed=bench.SEED, mode="fast")
        n = 1 << 22
        g = torch.Generator(device="cuda").manual_seed(1)
        x = torch.rand((n, 3), device="cuda", generator=g)
        w = torch.rand((n, 2), device="cuda", generator=g)
        gg = torch.zeros(n, device="cuda")
        res = torch.empty((n, 3), device="cuda")
        outs = {}
        for rep in range(2):
            for v in sys.argv[1].split(","):
                os.environ[VAR] = v
                ctx.load_field(fc, prm)
                sts = [ctx.render_neural(cam, rc, out=frame, stats=True)[1] for _ in range(8)][3:]
                for _ in range(2):
                    ctx.field_query(x, w, gg, out=res)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(5):
                    ctx.field_query(x, w, gg, out=res)
                b.record()
                torch.cuda.synchronize()
                outs[v] = res.cpu().numpy()
                print("wg", v, json.dumps({"ms_field_frame": float(np.mean([q["ms_field"] for q in sts])),
                                           "field_query_Mqps": n / (a.elapsed_time(b) / 5 / 1e3) / 1e6}), flush=True)
        k = list(outs)
        print("outputs identical:", bool(np.array_equal(outs[k[0]], outs[k[-1]])))
