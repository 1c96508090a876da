"""One config-3 KNN batch over a traced 4M-photon map with make_batch queries
(for ncu: -k regex:k_knn_query).  Tooling, not product."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import bench  # noqa: E402
import bench_knn  # noqa: E402
from paper_2304_07338_b200 import Context  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "traced"
r = float(sys.argv[2]) if len(sys.argv) > 2 else float("inf")
vol, tf, lights, cam = bench.scene_inputs()
with Context(0) as ctx:
    ctx.upload_volume(vol)
    ctx.set_medium(tf, 100.0)
    ctx.set_lights(lights)
    n, _ = bench_knn._build(ctx, kind, 32_000_000 if kind == "traced" else 4_000_000)
    x, w, g = bench_knn._train_queries(ctx, 1 << 20, 64)
    dt, mc = bench_knn._time_targets(ctx, x, w, g, 64, r, 1)
    print(kind, r, n, dt * 1e3, "ms", mc)
