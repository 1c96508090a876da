"""sha256 of one C2 frame (mode from argv) with the library PF_LIBPFGPU points at.
Tooling for A/B builds: a change that must not alter the frame compares hashes."""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2304_07338_b200 import Context, FieldConfig, RenderConfig  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "fast"
# optional: hold <GB> of device memory first (allocation placement must not change the frame)
import torch  # noqa: E402
_hold = torch.empty(int(float(sys.argv[2]) * 2**30), dtype=torch.uint8, device="cuda") if len(sys.argv) > 2 else None
vol, tf, lights, cam = bench.scene_inputs()
with Context(0) as ctx:
    ctx.upload_volume(vol)
    ctx.set_medium(tf, 100.0)
    ctx.set_lights(lights)
    fc = FieldConfig.paper()
    ctx.load_field(fc, fc.init_params(seed=bench.SEED, embed_scale=1e-2))
    rm = mode.replace("pt_", "")
    rc = RenderConfig(spp=bench.SPP, seed=bench.SEED, mode=rm)
    # "pt_fast" / "pt_parity": render_path_traced (its FAST walk shares the DDA)
    img = ctx.render_path_traced(cam, rc) if mode.startswith("pt_") else ctx.render_neural(cam, rc)
print(mode, hashlib.sha256(img.tobytes()).hexdigest()[:16], float(img.mean()))
