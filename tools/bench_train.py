"""Paper-scale field training throughput:
2^16 queries per step, K = 1024 KNN targets over a traced photon map, paper
photon field (16x8 hash grid, T = 2^19, 5x64 MLP).  Reports the device time
split between make_batch (KNN + Eq. 6/7) and train_step, per step.

  python tools/bench_train.py [--steps 30] [--photons 1000000] [--batch 65536] [--K 1024]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def run(ctx, steps=30, photons=1_000_000, batch=1 << 16, K=1024, fc=None):
    import numpy as np

    from paper_2304_07338_b200 import FieldConfig, TraceConfig, TrainConfig
    fc = fc or FieldConfig.paper()
    tc = TraceConfig(n_total=photons, seed=2)
    ctx.trace_photons(tc, device=True)
    ctx.knn_build_traced(tc.phase_set)
    ctx.train_init(fc, fc.init_params(seed=3, embed_scale=1e-4, bias_scale=0.0))
    # warm-up (allocations, module load)
    ctx.train(TrainConfig(total_steps=2, batch_size=batch, K=K, seed=1))
    res = ctx.train(TrainConfig(total_steps=steps, batch_size=batch, K=K, seed=5))
    return {"steps": steps, "batch": batch, "K": K, "photons_traced": photons,
            "ms_make_batch_per_step": res.knn_ms / steps, "ms_train_step_per_step": res.step_ms / steps,
            "train_queries_per_s": batch * steps / (res.step_ms * 1e-3),
            "loss_first_last": [float(res.loss_history[0]), float(res.loss_history[-1])],
            "finite": bool(np.all(np.isfinite(res.loss_history)))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--photons", type=int, default=1_000_000)
    ap.add_argument("--batch", type=int, default=1 << 16)
    ap.add_argument("--K", type=int, default=1024)
    a = ap.parse_args()
    from paper_2304_07338_b200 import Context
    from paper_2304_07338_b200.scene import default_lights, synth_volume, tf_scene_a
    ctx = Context(0)
    ctx.upload_volume(synth_volume("sphere_sinusoid", 256))
    ctx.set_medium(tf_scene_a(), 100.0)
    ctx.set_lights(default_lights())
    print(json.dumps(run(ctx, a.steps, a.photons, a.batch, a.K)))


if __name__ == "__main__":
    main()
