"""Diagnostics: FAST (DDA majorant) estimators vs PARITY.  Tooling, not product."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_07338_b200 import Context, FieldConfig, RenderConfig
from paper_2304_07338_b200.scene import CameraSpec, default_lights, synth_volume, tf_scene_a, tf_scene_b

with Context(0) as ctx:
    for tfn, tf in (("A", tf_scene_a()), ("B", tf_scene_b())):
        ctx.upload_volume(synth_volume("sphere_sinusoid", 64))
        ctx.set_medium(tf, 100.0)
        ctx.set_lights(default_lights())
        n = 400000
        r = np.random.default_rng(0)
        o = np.tile([0.5, 0.5, -0.9], (n, 1)) + 0.0
        d = np.column_stack([r.uniform(-0.3, 0.3, n), r.uniform(-0.3, 0.3, n), np.ones(n)])
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        idx = np.arange(n, dtype=np.uint64)
        hp, pp, _ = ctx.delta_track_batch(o, d, np.zeros(n), np.full(n, np.inf), 1, "camera", idx, fp64=True)
        hf, pf, _ = ctx.delta_track_batch(o, d, np.zeros(n), np.full(n, np.inf), 2, "camera", idx, fp64=False)
        print(tfn, "hit frac parity", hp.mean(), "fast", hf.mean(), "depth", pp[hp == 1, 2].mean(), pf[hf == 1, 2].mean())
        a = r.uniform(0.2, 0.8, (256, 3))
        b = np.tile([2.0, 2.5, -1.0], (256, 1))
        i2 = np.arange(256, dtype=np.uint64)
        tr = ctx.transmittance_batch(a, b, 3, "nee", i2, 4000, ratio=True)
        td = ctx.transmittance_batch(a, b, 4, "nee", i2, 4000)
        print(tfn, "T ratio-dda mean", tr.mean(), "delta", td.mean(), "max abs diff", np.abs(tr - td).max())
        cam = CameraSpec(64, 64)
        fc = FieldConfig.desk()
        ctx.load_field(fc, fc.init_params(seed=4, embed_scale=0.5, bias_scale=0.1))
        for name, kw in (("direct", dict(use_field=False)), ("field", dict(w_d=0.0)), ("both", {})):
            par = ctx.render_neural(cam, RenderConfig(spp=64, g=0.5, seed=1, mode="parity", **kw))
            fa = ctx.render_neural(cam, RenderConfig(spp=64, g=0.5, seed=1, mode="fast", **kw))
            print(tfn, name, "mean parity", par.mean(), "fast", fa.mean(), "rel rmse", np.sqrt(np.mean((fa - par) ** 2)) / par.mean())
