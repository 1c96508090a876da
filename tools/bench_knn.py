"""Config 3 microbench: KNN radiance targets (k=64) over a 4M-photon 3-phase map.
Device-resident queries/outputs, CUDA-event timed.  Tooling (bench.py reuses it)."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def run(ctx, n_photons=4_000_000, batch=1 << 20, K=64, reps=5, r_max=float("inf")):
    import torch
    from paper_2304_07338_b200._lib import check, lib
    from paper_2304_07338_b200.scene import synth_photons
    ph = synth_photons(n_photons, 3, seed=3)
    ph["power"] *= 1e-4
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    ctx.knn_build(ph, [-0.75, 0.0, 0.75])
    ev1.record()
    torch.cuda.synchronize()
    build_ms = ev0.elapsed_time(ev1)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.rand((batch, 3), device="cuda", generator=g)
    w = torch.nn.functional.normalize(torch.randn((batch, 3), device="cuda", generator=g, dtype=torch.float64), dim=1)
    gi = torch.randint(0, 3, (batch,), device="cuda", generator=g, dtype=torch.uint8)
    out = torch.empty((batch, 3), device="cuda", dtype=torch.float64)
    args = (ctx._h, batch, x.data_ptr(), w.data_ptr(), gi.data_ptr(), K, C.c_float(r_max), C.c_double(5.0),
            out.data_ptr(), None, None, None)
    for _ in range(2):
        check(lib().pf_knn_targets(*args))
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(reps):
        check(lib().pf_knn_targets(*args))
    ev1.record()
    torch.cuda.synchronize()
    dt = ev0.elapsed_time(ev1) / reps / 1e3
    return {"queries_per_s": batch / dt, "batch": batch, "K": K, "photons": n_photons, "ms_per_batch": dt * 1e3,
            "build_ms": build_ms, "algorithmic_GBps": batch * K * 40 / dt / 1e9}


if __name__ == "__main__":
    from paper_2304_07338_b200 import Context
    import torch
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    with Context(0, stream=s.cuda_stream) as ctx:
        print(json.dumps(run(ctx)))
