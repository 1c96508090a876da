"""SPEC acceptance criteria 6-10 on the GPU pipeline:
trace (Alg. 1) -> staggered training -> neural / photon-map / path-traced
renders of the 64^3 synthetic slab.  Prints one JSON report; the GPU tests
(tests/test_gpu_acceptance.py) assert on the same quantities."""
from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from paper_2304_07338_b200 import (FieldConfig, PathTraceConfig, RenderConfig, TraceConfig,  # noqa: E402
                                   TrainConfig)
from paper_2304_07338_b200.imaging import luminance, rse  # noqa: E402
from paper_2304_07338_b200.imaging import ssim as _ssim  # noqa: E402


def ssim(a, ref):
    """SSIM on linear radiance with the reference image's luminance range as L."""
    return _ssim(a, ref, data_range=float(luminance(ref).max()))
from paper_2304_07338_b200.scene import CameraSpec, default_lights, synth_volume  # noqa: E402

# slab: sigma_t = density 5 x alpha 1 inside (optical depth 1.25 across), albedo 0.9 -> strong
# multiple scattering, so L_i matters next to L_d
SLAB_TF = np.array([[0.0, 0.9, 0.9, 0.9, 0.0], [1.0, 0.9, 0.9, 0.9, 1.0]])
SLAB_DENSITY = 5.0
PHASES = [-0.75, 0.0, 0.75]
CAM = CameraSpec(64, 64)


def setup(ctx, photons=1_000_000, phases=PHASES, seed=2):
    ctx.upload_volume(synth_volume("slab", 64))
    ctx.set_medium(SLAB_TF, SLAB_DENSITY)
    ctx.set_lights(default_lights())
    tc = TraceConfig(n_total=photons, phase_set=list(phases), seed=seed)
    ctx.trace_photons(tc, device=True)
    ctx.knn_build_traced(phases)


def train(ctx, steps=1500, K=256, ends=(0.36, 0.63, 0.90, 1.0), radii=(0.25, 0.5, 2.5, 5.0), seed=4):
    fc = FieldConfig.desk()
    ctx.train_init(fc, fc.init_params(seed=3, embed_scale=1e-4, bias_scale=0.0))
    return ctx.train(TrainConfig(total_steps=steps, batch_size=4096, K=K, schedule_ends=ends,
                                 schedule_radii=radii, seed=seed))


def render_pair(ctx, g, spp=16, seed=1, K=256, r_max=5.0, w_d=1.0):
    rc = RenderConfig(spp=spp, g=g, seed=seed, mode="fast", w_d=w_d)
    return ctx.render_neural(CAM, rc), ctx.render_photon_map(CAM, rc, K=K, r_max=r_max)


def lum_var(frames):
    return float(np.mean(np.var(np.stack([luminance(f) for f in frames]), axis=0)))


def rel_var(frames):
    """Noise relative to signal: mean per-pixel luminance variance / mean luminance^2."""
    lum = np.stack([luminance(f) for f in frames])
    return float(np.mean(np.var(lum, axis=0)) / np.mean(lum) ** 2)


def run(ctx):
    rep = {}
    setup(ctx)
    res = train(ctx)
    rep["train_loss_first_last"] = [float(res.loss_history[0]), float(np.median(res.loss_history[-20:]))]
    # 7. reconstruction fidelity (full compose, and the in-scattered term alone)
    nf, pm = render_pair(ctx, 0.0)
    nfi, pmi = render_pair(ctx, 0.0, w_d=0.0)
    rep["A7_ssim"] = ssim(nf, pm)
    rep["A7_ssim_Li_only"] = ssim(nfi, pmi)
    rep["A7_mean_rse"] = float(np.mean(rse(nf, pm)))
    # 8. noise ordering: 16 independent 1-spp renders, per-pixel luminance variance
    neu = [ctx.render_neural(CAM, RenderConfig(spp=1, g=0.0, seed=100 + s, mode="fast")) for s in range(16)]
    pt1 = [ctx.render_path_traced(CAM, RenderConfig(spp=1, g=0.0, seed=200 + s, mode="fast"), PathTraceConfig())
           for s in range(16)]
    pt4 = [ctx.render_path_traced(CAM, RenderConfig(spp=4, g=0.0, seed=300 + s, mode="fast"), PathTraceConfig())
           for s in range(16)]
    rep["A8_var_neural_1spp"], rep["A8_var_pt_1spp"], rep["A8_var_pt_4spp"] = lum_var(neu), lum_var(pt1), lum_var(pt4)
    rep["A8_relvar_neural_1spp"], rep["A8_relvar_pt_1spp"], rep["A8_relvar_pt_4spp"] = rel_var(neu), rel_var(pt1), rel_var(pt4)
    rep["A8_mean_lum"] = [float(np.mean([luminance(f).mean() for f in x])) for x in (neu, pt1)]
    li_n = [ctx.render_neural(CAM, RenderConfig(spp=1, g=0.0, seed=100 + s, mode="fast", w_d=0.0)) for s in range(16)]
    li_p = [ctx.render_path_traced(CAM, RenderConfig(spp=1, g=0.0, seed=200 + s, mode="fast", w_d=0.0), PathTraceConfig())
            for s in range(16)]
    rep["A8_Li_mean_neural_pt"] = [float(np.mean([luminance(f).mean() for f in x])) for x in (li_n, li_p)]
    # 9. cost scaling: path tracer time grows with max_bounces, neural has no such parameter
    ctx.set_timing(True)
    big = CameraSpec(512, 512)
    t_pt = {}
    for mb in (2, 4, 8, 16):
        sts = [ctx.render_path_traced(big, RenderConfig(spp=8, g=0.0, seed=5, mode="fast"), PathTraceConfig(max_bounces=mb),
                                      stats=True)[1] for _ in range(4)]
        t_pt[mb] = float(np.median([s["ms_trace"] for s in sts[1:]]))
    sts = [ctx.render_neural(big, RenderConfig(spp=8, g=0.0, seed=5, mode="fast"), stats=True)[1] for _ in range(4)]
    rep["A9_pt_trace_ms"] = t_pt
    rep["A9_neural_ms"] = float(np.median([s["ms_trace"] + s["ms_field"] for s in sts[1:]]))
    ctx.set_timing(False)
    # 10. phase generalisation: trained on G = {-0.75, 0, 0.75}; unseen g = +-0.35 vs maps traced at those g
    trained = [ssim(*render_pair(ctx, g)) for g in PHASES]
    field_unseen = {g: ctx.render_neural(CAM, RenderConfig(spp=16, g=g, seed=1, mode="fast")) for g in (-0.35, 0.35)}
    setup(ctx, phases=[-0.35, 0.35], seed=7)
    unseen = [ssim(field_unseen[g], ctx.render_photon_map(CAM, RenderConfig(spp=16, g=g, seed=1, mode="fast"),
                                                          K=256, r_max=5.0)) for g in (-0.35, 0.35)]
    rep["A10_ssim_trained_g"], rep["A10_ssim_unseen_g"] = trained, unseen
    return rep


if __name__ == "__main__":
    from paper_2304_07338_b200 import Context
    with Context(0) as ctx:
        print(json.dumps(run(ctx)))
