"""Small config-1-style workload for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel family once -- parity + fast render with the field,
path tracer, photon map (trace + KNN build + query + targets), one train step."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from paper_2304_07338_b200 import (Context, FieldConfig, PathTraceConfig, RenderConfig,  # noqa: E402
                                   TraceConfig)
from paper_2304_07338_b200.scene import CameraSpec, default_lights, synth_volume, tf_scene_b  # noqa: E402

with Context(0) as ctx:
    ctx.upload_volume(synth_volume("sphere_sinusoid", 32))
    ctx.set_medium(tf_scene_b(), 100.0)
    ctx.set_lights(default_lights())
    fc = FieldConfig.desk()
    p = fc.init_params(seed=1, embed_scale=0.3, bias_scale=0.1)
    ctx.load_field(fc, p)
    cam = CameraSpec(48, 32)
    for mode in ("parity", "fast"):
        ctx.render_neural(cam, RenderConfig(spp=1, seed=1, mode=mode))
        ctx.render_path_traced(cam, RenderConfig(spp=1, seed=1, mode=mode), PathTraceConfig(max_bounces=4))
    tc = TraceConfig(n_total=20000, seed=2)
    ctx.trace_photons(tc, device=True)
    ctx.knn_build_traced(tc.phase_set)
    ctx.render_photon_map(cam, RenderConfig(spp=1, seed=1, mode="fast"), K=16)
    r = np.random.default_rng(0)
    x = r.random((256, 3)).astype(np.float32)
    g = r.integers(0, 3, 256).astype(np.uint8)
    ctx.knn_query(x, g, 32)
    ctx.knn_query(x, g, 200)
    w = r.standard_normal((256, 3))
    w /= np.linalg.norm(w, axis=1, keepdims=True)
    ctx.knn_targets(x, w, g, 32)
    ctx.train_init(fc, p)
    ctx.train_step(x, r.random((256, 2)).astype(np.float32), np.zeros(256, np.float32),
                   r.random((256, 3)).astype(np.float32), 0, 10)
    ctx.synchronize()
print("sanitize workload done")
