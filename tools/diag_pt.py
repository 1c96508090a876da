import numpy as np
from paper_2304_07338_b200 import Context, PathTraceConfig, RenderConfig
from paper_2304_07338_b200.scene import CameraSpec, default_lights, synth_volume, tf_scene_b
ctx = Context(0)
ctx.upload_volume(synth_volume("sphere_sinusoid", 48)); ctx.set_medium(tf_scene_b(), 100.0); ctx.set_lights(default_lights())
cam = CameraSpec(80, 60)
rc = RenderConfig(spp=2, g=-0.3, seed=3, mode="fast", use_field=False, background=(0.3, 0.2, 0.1))
a = ctx.render_path_traced(cam, rc, PathTraceConfig(max_bounces=1)).astype(np.float64)
b = ctx.render_neural(cam, rc).astype(np.float64)
d = np.abs(a-b); bad = np.any(d > 0, axis=2)
print("n diff px", bad.sum(), "max abs", d.max(), "max rel", (d/np.maximum(np.abs(b),1e-30)).max(), "mean", a.mean(), b.mean())
idx = np.argwhere(bad)[:5]
for y,x in idx: print(y,x,a[y,x],b[y,x])
