"""Config 3 microbench: KNN radiance targets (k=64) over 4M-photon 3-phase maps.

Inputs follow SURVEY 8(d): queries from make_batch's generator (x ~ U^3,
omega ~ sphere, g ~ U(G) on Stream::Train), three maps
(uniform and clustered synthetic 4M-photon maps, and a map traced through the
bench scene by the GPU photon tracer), r_max in {inf, 0.05, 0.25}.
Device-resident queries/outputs, CUDA-event timed.  Tooling (bench.py reuses it).
"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

RADII = (float("inf"), 0.05, 0.25)


def _train_queries(ctx, batch, K, seed=11):
    """make_batch's queries (Stream::Train, step 0) into device buffers."""
    import torch
    from paper_2304_07338_b200._lib import check, lib
    x = torch.empty((batch, 3), device="cuda", dtype=torch.float32)
    w = torch.empty((batch, 3), device="cuda", dtype=torch.float64)
    g = torch.empty((batch,), device="cuda", dtype=torch.uint8)
    t = torch.empty((batch, 3), device="cuda", dtype=torch.float64)
    check(lib().pf_make_batch(ctx._h, seed, 0, batch, K, C.c_float(float("inf")), C.c_double(5.0),
                              x.data_ptr(), w.data_ptr(), g.data_ptr(), t.data_ptr()))
    return x, w, g


def _time_targets(ctx, x, w, g, K, r_max, reps):
    import torch
    from paper_2304_07338_b200._lib import check, lib
    batch = x.shape[0]
    out = torch.empty((batch, 3), device="cuda", dtype=torch.float64)
    cnt = torch.empty((batch,), device="cuda", dtype=torch.int32)
    ids = torch.empty((batch, K), device="cuda", dtype=torch.int32)
    d2 = torch.empty((batch, K), device="cuda", dtype=torch.float32)
    # one untimed call with the id/count outputs (the counts give the bytes
    # actually gathered when r_max cuts the list short)
    check(lib().pf_knn_targets(ctx._h, batch, x.data_ptr(), w.data_ptr(), g.data_ptr(), K, C.c_float(r_max),
                               C.c_double(5.0), out.data_ptr(), ids.data_ptr(), d2.data_ptr(), cnt.data_ptr()))
    args = (ctx._h, batch, x.data_ptr(), w.data_ptr(), g.data_ptr(), K, C.c_float(r_max), C.c_double(5.0),
            out.data_ptr(), None, None, None)
    for _ in range(2):
        check(lib().pf_knn_targets(*args))
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(reps):
        check(lib().pf_knn_targets(*args))
    ev1.record()
    torch.cuda.synchronize()
    dt = ev0.elapsed_time(ev1) / reps / 1e3
    mean_count = float(cnt.double().mean().item())
    return dt, mean_count


def _build(ctx, kind, n_photons):
    import torch
    from paper_2304_07338_b200.scene import synth_photons
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if kind == "traced":
        from paper_2304_07338_b200.api import TraceConfig
        tc = TraceConfig(n_total=n_photons, seed=5)
        tr = ctx.trace_photons(tc, device=True)
        n = int(tr.photons.shape[0])
        torch.cuda.synchronize()
        ev0.record()
        ctx.knn_build(tr.photons, tc.phase_set)
        ev1.record()
        del tr
    else:
        ph = synth_photons(n_photons, 3, seed=3, clustered=(kind == "clustered"))
        ph["power"] *= 1e-4
        n = len(ph)
        torch.cuda.synchronize()
        ev0.record()
        ctx.knn_build(ph, [-0.75, 0.0, 0.75])
        ev1.record()
    torch.cuda.synchronize()
    return n, ev0.elapsed_time(ev1)


def run(ctx, n_photons=4_000_000, batch=1 << 20, K=64, reps=5, maps=("uniform", "clustered", "traced"),
        radii=RADII, hbm_gbs=None):
    """Headline = uniform map, r_max = inf (every query gathers K records);
    'matrix' holds every (map, r_max) cell with its own roofline."""
    x = w = g = None
    cells = []
    for kind in maps:
        # the traced map needs the scene uploaded by the caller: the bench scene
        # deposits ~0.12 photons per emitted one, so 8x emitted gives ~4M deposits
        n, build_ms = _build(ctx, kind, n_photons if kind != "traced" else 8 * n_photons)
        if x is None:  # make_batch needs a built map; the same queries serve every map (3 phases each)
            x, w, g = _train_queries(ctx, batch, K)
        for r in radii:
            dt, mc = _time_targets(ctx, x, w, g, K, r, reps)
            alg = batch * K * 40 / dt / 1e9
            got = batch * mc * 40 / dt / 1e9
            c = {"map": kind, "photons": n, "r_max": r if r != float("inf") else "inf", "queries_per_s": batch / dt,
                 "ms_per_batch": dt * 1e3, "mean_found": mc, "build_ms": build_ms,
                 "algorithmic_GBps": alg, "gathered_GBps": got}
            if hbm_gbs:
                c["roofline"] = {"bound": "hbm", "achieved": alg, "peak": hbm_gbs, "unit": "GB/s",
                                 "frac": alg / hbm_gbs, "frac_gathered": got / hbm_gbs}
            cells.append(c)
    head = next((c for c in cells if c["map"] == maps[0] and c["r_max"] == "inf"), cells[0])
    return {"queries_per_s": head["queries_per_s"], "batch": batch, "K": K, "photons": head["photons"],
            "map": head["map"], "r_max": head["r_max"], "ms_per_batch": head["ms_per_batch"],
            "build_ms": head["build_ms"], "algorithmic_GBps": head["algorithmic_GBps"],
            "queries": "make_batch generator: Stream::Train, step 0 (x ~ U^3, omega ~ sphere, g ~ U(G))",
            "matrix": cells}


if __name__ == "__main__":
    import bench
    from paper_2304_07338_b200 import Context
    import torch
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    vol, tf, lights, cam = bench.scene_inputs()
    with Context(0, stream=s.cuda_stream) as ctx:
        ctx.upload_volume(vol)
        ctx.set_medium(tf, 100.0)
        ctx.set_lights(lights)
        print(json.dumps(run(ctx, hbm_gbs=float(bench.load_peaks()[0]["hbm_gbs"]))))
