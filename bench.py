#!/usr/bin/env python
"""Headline benchmark: neural photon-field rendering, BASELINE config 2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full frame of render_neural (Alg. 2): 1920x1080, 8 spp, 256^3
synthetic volume, one point light, paper-size photon field (16x8 hash grid,
T = 2^19, 5x64 MLP).  The headline is PARITY mode: the reference's own
estimator (binary64 delta tracking against the global majorant, delta-trial
NEE, the reference's RNG consumption; proj/src/volume.cpp:204-256), so
value / e2e compare like-for-like with `--impl reference`, the unmodified
reference CPU path on the host cores.  FAST mode (binary32, macro-cell DDA +
ratio tracking, statistically equivalent) is reported under "fast".
N > 1: image tiles are interleaved over the ranks (strong scaling of one
frame) and gathered to rank 0.  Timing: W untimed warm-up frames, then K
frames, each bracketed by CUDA events on the render stream with an L2 flush
(256 MiB write) between frames; barrier + synchronize around the timed
region; the max over ranks is reported.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
# BASELINE.json configs: c2 is the headline (fits one GPU); c4 / c5 are the
# multi-GPU shapes, runnable here on N >= 1 GPUs with --config.
CONFIGS = {
    "c2": dict(W=1920, H=1080, spp=8, vol=256, dynamic=False,
               desc="config 2: 256^3 sphere_sinusoid volume (scene A TF, density 100), 1920x1080, 8 spp"),
    "c4": dict(W=3840, H=2160, spp=16, vol=512, dynamic=False,
               desc="config 4: 512^3 sphere_sinusoid volume (scene A TF, density 100), 3840x2160, 16 spp"),
    "c5": dict(W=1920, H=1080, spp=8, vol=1024, dynamic=True,
               desc="config 5: 1024^3 sphere_sinusoid volume, 1920x1080, 8 spp, transfer function and "
                    "light changed every frame (majorant grid rebuilt per frame)"),
}
W_, H_, SPP, VOL_N, SEED = 1920, 1080, 8, 256, 2024
METRIC = "frames/s at 1920x1080, 8 spp, 256^3 volume (neural render, Alg. 2)"
CFG = CONFIGS["c2"]


def select_config(name: str) -> None:
    global W_, H_, SPP, VOL_N, METRIC, CFG
    CFG = CONFIGS[name]
    W_, H_, SPP, VOL_N = CFG["W"], CFG["H"], CFG["spp"], CFG["vol"]
    METRIC = f"frames/s at {W_}x{H_}, {SPP} spp, {VOL_N}^3 volume (neural render, Alg. 2)"


def dynamic_scene(i: int, tf0, lights0):
    """Config 5: per-frame transfer function (alpha ramp scaled) and orbiting light."""
    import math
    tf = tf0.copy()
    tf[:, 4] = np.clip(tf0[:, 4] * (0.75 + 0.25 * math.cos(0.37 * i)), 0.0, 1.0)
    li = lights0.copy()
    a = 0.21 * i
    li[0, 0], li[0, 2] = 0.5 + 2.0 * math.cos(a), 0.5 + 2.0 * math.sin(a)
    return tf, li


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def scene_inputs():
    from paper_2304_07338_b200.scene import CameraSpec, default_lights, synth_volume, tf_scene_a
    return synth_volume("sphere_sinusoid", VOL_N), tf_scene_a(), default_lights(), CameraSpec(W_, H_)


class ClockSampler:
    """nvidia-smi-equivalent clocks sampling (NVML) during the timed region."""

    def __init__(self, dev: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {getattr(nv, k, None): v for k, v in [
            ("nvmlClocksEventReasonHwSlowdown", "hw_slowdown"),
            ("nvmlClocksEventReasonHwThermalSlowdown", "hw_thermal_slowdown"),
            ("nvmlClocksEventReasonSwThermalSlowdown", "sw_thermal_slowdown"),
            ("nvmlClocksEventReasonSwPowerCap", "sw_power_cap"),
            ("nvmlClocksEventReasonHwPowerBrakeSlowdown", "hw_power_brake_slowdown")] if getattr(nv, k, None)}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.01)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------ reference ----

def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def reference_inputs():
    """Config-2 inputs for the reference CPU path WITHOUT the GPU library: the
    paper field's parameters come from the oracle's restatement of
    pf_field_init (same draw order, tests/test_host.py pins the equality)."""
    from types import SimpleNamespace as NS

    from oracle import oracle as o
    vol, tf, lights, cam = scene_inputs()
    fc = NS(pos=NS(dims=3, levels=16, features=8, base_res=4, growth=2.0, log2_table=19),
            dir=NS(dims=2, levels=16, features=8, base_res=4, growth=2.0, log2_table=19),
            hidden_layers=5, width=64, psi=5.0)
    params = o.field_init(fc, seed=SEED, embed_scale=1e-2, bias_scale=0.0)
    rc = NS(spp=SPP, g=0.0, seed=SEED, w_d=1.0, w_i=1.0, background=(0.0, 0.0, 0.0), nee_trials=1,
            use_field=True)
    return vol, tf, lights, cam, fc, params, rc


def reference_cpu_frame(sc, lights, fc, params, cam_spec, rc, workers: int) -> tuple[float, int]:
    """One WHOLE frame of the reference CPU render path: pf::delta_track +
    pf::transmittance (proj/src/volume.cpp:204-256, compiled unmodified in
    oracle/_ref) driven by pf::parallel_chunks in chunks of 4096 samples
    (proj/src/parallel.cpp:22-49) on `workers` host threads, with the SPEC-only
    pieces (camera, NEE term, binary64 field forward, compose) from the C
    restatement.  Returns (seconds, hits)."""
    from oracle import oracle as o
    t0 = time.perf_counter()
    if isinstance(sc, o.RefScene):
        _, st = o.ref_render_neural(sc, lights, fc, params, cam_spec, rc, workers=workers)
    else:  # no oracle/_ref on this host: the single-threaded C restatement ("port")
        _, st = o.render_neural(sc, lights, fc, params, cam_spec, rc)
    return time.perf_counter() - t0, int(st["hits"])


def cpu_baseline_kind():
    from oracle import oracle as o
    return "reference" if o.ref_available() else "port"


def run_reference(args):
    """--impl reference: the reference's own CPU path timed on the host cores,
    whole config-2 frames (median of --steps frames after --warmup frames)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as o
    workers = os.cpu_count() or 1
    kind = "reference" if o.ref_available() else "port"
    vol, tf, lights, cam, fc, params, rc = reference_inputs()
    sc = o.RefScene(vol, tf, 100.0) if kind == "reference" else o.OracleScene(vol, tf, 100.0)
    t_wall0 = time.perf_counter()
    for _ in range(args.warmup):
        reference_cpu_frame(sc, lights, fc, params, cam, rc, workers)
    res = [reference_cpu_frame(sc, lights, fc, params, cam, rc, workers) for _ in range(args.steps)]
    wall = time.perf_counter() - t_wall0
    sec = float(np.median([r[0] for r in res]))
    fps = 1.0 / sec
    sample = (f"whole frames: {W_}x{H_} px x {SPP} spp = {W_ * H_ * SPP} samples per step, median of "
              f"{args.steps} frames after {args.warmup} warm-up frames; pf::delta_track + pf::transmittance "
              f"(unmodified volume.cpp) via pf::parallel_chunks(chunk 4096 samples) + binary64 field forward")
    line = {"metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": CFG["desc"] + ", 1 point light, paper photon field (random init)",
                       "mode": "parity", "cpu": f"{cpu_model()}, {workers} threads"},
            "frame": {"samples": W_ * H_ * SPP, "hits": res[0][1],
                      "sec_min": float(np.min([r[0] for r in res])),
                      "sec_max": float(np.max([r[0] for r in res])), "wall_s": wall},
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": workers, "kind": kind,
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ ours ----

def trace_kernel_name(mode: str) -> str:
    return "k_render_trace_fast" if mode == "fast" else "k_render_trace_parity"


def load_traffic():
    tfile = ROOT / "profiles" / "traffic.json"
    return json.loads(tfile.read_text()) if tfile.exists() else {}


def roofline_for(mode: str, stats: list, peaks, peak_kind: str, traffic: dict) -> dict:
    """HBM roofline of the dominant kernel (the tracer) per SURVEY 8(d): 32 B
    (8 x f32 voxels) per voxel fetch actually issued (PARITY skips the fetch of
    every certain-null collision; FAST fetches at every tentative collision of
    its macro-cell DDA), over the tracer's CUDA-event time on the render stream.
    The tracers are issue-bound, so ncu's issue / FP64 pipe / lane figures for
    the same kernel (profiles/, cold cache) ride along."""
    kname = trace_kernel_name(mode)
    tr_ms = float(np.mean([s["ms_trace"] for s in stats]))
    steps = float(np.mean([s["primary_steps"] + s["shadow_steps"] for s in stats]))
    fetches = float(np.mean([s["voxel_fetches"] for s in stats]))
    hbm = float(peaks["hbm_gbs"])
    achieved = fetches * 32.0 / (tr_ms * 1e-3) / 1e9
    k = traffic.get("kernels", {}).get(kname, {})
    return {"kernel": kname, "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": k.get("dram_bytes"),
            "per_unit": f"32 B (8 x f32 voxels) per voxel fetch issued, {fetches:.4g} fetches per launch "
                        f"({steps:.4g} tentative collisions)",
            "peak_source": peak_kind,
            "tentative_collisions_per_s": steps / (tr_ms * 1e-3),
            "issue": {"sm_issue_active_pct": k.get("sm_issue_active_pct"),
                      "fp64_pipe_pct": k.get("fp64_pipe_pct"),
                      "lane_efficiency": k.get("lane_efficiency"),
                      "source": traffic.get("source")}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="parity", choices=["fast", "parity"],
                    help="headline mode (parity = the reference's binary64 estimator)")
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-fast", action="store_true", help="skip the FAST-mode extra line")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    select_config(args.config)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2304_07338_b200 import Context, FieldConfig, RenderConfig
    from paper_2304_07338_b200 import build as pfbuild

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # smoke-testing the N > 1 logic on a 1-GPU box: PF_BENCH_ONE_DEVICE=1 puts
    # every rank on cuda:0 and PF_DIST_BACKEND=gloo (NCCL refuses duplicate GPUs)
    if os.environ.get("PF_BENCH_ONE_DEVICE") == "1":
        local = 0
    if world > 1:
        backend = os.environ.get("PF_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    if not (ROOT / "paper_2304_07338_b200" / "libpfgpu.so").exists():
        if rank == 0:
            pfbuild.build()
        if world > 1:
            dist.barrier()

    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = Context(local, stream=stream.cuda_stream)
    vol, tf, lights, cam_spec = scene_inputs()
    ctx.upload_volume(vol)
    ctx.set_medium(tf, 100.0)
    ctx.set_lights(lights)
    fc = FieldConfig.paper()
    params = fc.init_params(seed=SEED, embed_scale=1e-2, bias_scale=0.0)
    ctx.load_field(fc, params)
    cam = ctx.camera(cam_spec)

    def rconf(mode):
        return RenderConfig(spp=SPP, g=0.0, seed=SEED, mode=mode, use_field=True, tile=(16, 16),
                            shard_index=rank, shard_count=world)

    rc = rconf(args.mode)
    frame = torch.zeros((H_, W_, 3), dtype=torch.float32, device="cuda")
    n_tiles_max = max(ctx.tiles_count(cam, rc, s) for s in range(world))
    per_shard = n_tiles_max * 16 * 16 * 3
    packed = torch.zeros(per_shard, dtype=torch.float32, device="cuda")
    gathered = torch.zeros(per_shard * world, dtype=torch.float32, device="cuda") if world > 1 else None
    # N > 1 tile gather: "p2p" = every rank's compose kernel stores its tiles
    # straight into rank 0's frame over NVLink (CUDA IPC mapping), fenced by a
    # stream-ordered 1-element all-reduce; "nccl" = pack / all_gather / unpack.
    gather = os.environ.get("PF_GATHER", "p2p") if world > 1 else "none"
    sync = torch.zeros(1, dtype=torch.float32, device="cuda")
    if gather == "p2p":
        ok = 1
        try:
            obj = [None]
            if rank == 0:
                shared, obj[0] = ctx.ipc_frame_create(H_, W_)
            dist.broadcast_object_list(obj, src=0)
            if rank != 0:
                shared = ctx.ipc_frame_open(obj[0], H_, W_)
        except Exception as e:  # no IPC / peer access on this box: NCCL gather instead
            print(f"rank {rank}: p2p gather unavailable ({e}); using NCCL", file=sys.stderr)
            ok = 0
        t = torch.tensor([ok], dtype=torch.int32, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if int(t.item()) == 1:
            frame = shared
        else:
            gather = "nccl"
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    ctx.set_timing(True)
    frame_no = [0]

    def step(rc_, stats=True):
        if CFG["dynamic"]:  # config 5: new TF + light every frame
            tf_i, li_i = dynamic_scene(frame_no[0], tf, lights)
            ctx.set_medium(tf_i, 100.0)
            ctx.set_lights(li_i)
        frame_no[0] += 1
        if gather == "p2p":
            dist.all_reduce(sync)  # rank 0 is done with the previous frame
        st = ctx.render_neural(cam, rc_, out=frame, stats=stats)
        if gather == "p2p":
            dist.all_reduce(sync)  # every rank's tiles are in rank 0's frame
        elif gather == "nccl":
            ctx.tiles_pack(cam, rc_, frame, packed)
            if dist.get_backend() == "nccl":
                dist.all_gather_into_tensor(gathered, packed)
            else:  # gloo (the one-GPU smoke test of this path): list all_gather
                dist.all_gather(list(gathered.view(world, -1).unbind(0)), packed)
            if rank == 0:
                ctx.tiles_unpack(cam, rc_, gathered, per_shard, frame)
        return st[1] if stats else None

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def time_frames(rc_):
        """W warm-up frames, then K frames each bracketed by CUDA events on the
        render stream, L2 flushed (256 MiB write, untimed) before each."""
        for _ in range(args.warmup):
            step(rc_)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        stats = []
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            t_wall0 = time.perf_counter()
            for i in range(args.steps):
                flush.fill_(float(i))
                ev[i][0].record()
                stats.append(step(rc_))
                ev[i][1].record()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            wall = time.perf_counter() - t_wall0
        total_ms = max_over_ranks(float(np.sum([a.elapsed_time(b) for a, b in ev])))
        return total_ms / args.steps, stats, clk.summary(), wall

    def time_e2e(rc_):
        """The public API with HOST buffers: per-frame TF + lights in, the frame
        out to pinned host memory, host<->device copies inside the timed region."""
        host_frame = torch.empty((H_, W_, 3), dtype=torch.float32, pin_memory=True)
        # per-frame TF + lights: config 5's animation (the same scenes the device-
        # timed loop renders), else the fixed scene re-sent every frame
        scenes = [dynamic_scene(frame_no[0] + i, tf, lights) if CFG["dynamic"] else (tf, lights)
                  for i in range(args.steps)]
        tf_hs = [torch.from_numpy(np.ascontiguousarray(a).copy()).pin_memory() for a, _ in scenes]
        li_hs = [torch.from_numpy(np.ascontiguousarray(b).copy()).pin_memory() for _, b in scenes]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        if world == 1:
            # pipelined: frame i's device->host copy overlaps frame i+1's kernels
            # (pf_render_neural_async); every frame is read back before the loop ends
            hosts = [host_frame, torch.empty_like(host_frame).pin_memory()]
            for i in range(3):
                ctx.render_neural_async(cam, rc_, hosts[i % 2].numpy())
            ctx.synchronize()
            t0 = time.perf_counter()
            for i in range(args.steps):
                ctx.set_medium(tf_hs[i].numpy(), 100.0)
                ctx.set_lights(li_hs[i].numpy())
                ctx.render_neural_async(cam, rc_, hosts[i % 2].numpy())
                if i > 0:
                    ctx.frame_wait(hosts[(i - 1) % 2].numpy())
            ctx.frame_wait(hosts[(args.steps - 1) % 2].numpy())
            e_ms = (time.perf_counter() - t0) / args.steps * 1e3
        else:
            times = []
            for i in range(args.steps):
                t0 = time.perf_counter()
                ctx.set_medium(tf_hs[i].numpy(), 100.0)
                ctx.set_lights(li_hs[i].numpy())
                step(rc_, stats=False)
                if rank == 0:
                    host_frame.copy_(frame, non_blocking=True)
                torch.cuda.synchronize()
                times.append(time.perf_counter() - t0)
            e_ms = float(np.mean(times)) * 1e3
        e_ms = max_over_ranks(e_ms)
        h2d = tf.nbytes + lights.nbytes + 104 + 128   # TF + lights + camera + render desc
        return {"value": 1000.0 / e_ms, "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(H_ * W_ * 12) if rank == 0 else 0}

    peaks, peak_kind = load_peaks()
    traffic = load_traffic()

    def frame_summary(stats, wall):
        hits = float(np.mean([s["hits"] for s in stats]))
        samples = float(np.mean([s["samples"] for s in stats]))
        steps = float(np.mean([s["primary_steps"] + s["shadow_steps"] for s in stats]))
        return {"samples": samples * world, "hits": hits, "hit_fraction": hits / max(samples, 1),
                "steps_per_sample": steps / max(samples, 1),
                "voxel_fetches": float(np.mean([s["voxel_fetches"] for s in stats])),
                "ms_trace": float(np.mean([s["ms_trace"] for s in stats])),
                "ms_field": float(np.mean([s["ms_field"] for s in stats])),
                "ms_compose": float(np.mean([s["ms_compose"] for s in stats])), "wall_s": wall}

    # ---- headline: the reference's estimator (PARITY, binary64) unless --mode fast
    ms_per_step, stats, clocks, wall = time_frames(rc)
    fps = 1000.0 / ms_per_step
    samples = float(np.mean([s["samples"] for s in stats]))
    e2e = time_e2e(rc)
    launches = int(sum(s["kernel_launches"] for s in stats)) + (2 * args.steps if gather == "nccl" else 0)

    # ---- FAST mode (binary32, macro-cell DDA + ratio-tracked NEE) as an extra
    fast = None
    if args.mode == "parity" and not args.no_fast:
        rcf = rconf("fast")
        f_ms, f_stats, f_clk, f_wall = time_frames(rcf)
        fast = {"value": 1000.0 / f_ms, "unit": "frames/s", "ms_per_step": f_ms, "dtype": "f32",
                "note": "binary32 delta tracking against macro-cell majorants + ratio-tracked shadow rays: "
                        "a different, unbiased estimator (statistical parity with the reference, "
                        "tests/test_gpu_c2.py); NOT the headline",
                "mrays_per_s": samples * world / (f_ms * 1e-3) / 1e6,
                "frame": frame_summary(f_stats, f_wall),
                "roofline": roofline_for("fast", f_stats, peaks, peak_kind, traffic),
                "e2e": time_e2e(rcf), "clocks": f_clk,
                "gpu_launches": int(sum(s["kernel_launches"] for s in f_stats))}

    # ---- extras (every rank runs its own query shard; rank 0 reports the aggregate)
    extras = {}
    if not args.no_extras:
        extras = bench_extras(ctx, fc, params, peaks, rank, world, cam=cam, rc=rc, frame=frame)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:  # the reference CPU path: 3 whole frames on the host cores, median
            from oracle import oracle as o
            workers = os.cpu_count() or 1
            rvol, rtf, rlights, rcam, rfc, rparams, rrc = reference_inputs()
            kind = cpu_baseline_kind()
            sc = o.RefScene(rvol, rtf, 100.0) if kind == "reference" else o.OracleScene(rvol, rtf, 100.0)
            ts = [reference_cpu_frame(sc, rlights, rfc, rparams, rcam, rrc, workers)[0] for _ in range(3)]
            cpu = {"value": 1.0 / float(np.median(ts)), "unit": "frames/s", "cores": workers, "kind": kind,
                   "cpu_model": cpu_model(),
                   "sample": f"3 whole frames ({W_ * H_ * SPP} samples each), median {np.median(ts):.2f} s; "
                             f"unmodified pf::delta_track/transmittance via parallel_chunks(4096) + "
                             f"binary64 field"}
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": "frames/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {e}"}

    dump = os.environ.get("PF_BENCH_DUMP")  # tests: rank 0 saves the last headline frame
    if dump:
        step(rc, stats=False)
        torch.cuda.synchronize()
        if rank == 0:
            np.save(dump, frame.cpu().numpy())
    if rank == 0:
        line = {
            "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if args.mode == "fast" else "f64", "data": "synthetic",
            "config": {"workload": CFG["desc"] + ", 1 point light, paper photon field "
                                                 "(16x8 hash grid T=2^19, 5x64 MLP, random init)",
                       "mode": args.mode,
                       "estimator": ("reference: binary64 delta tracking with the global majorant, "
                                     "delta-trial NEE, the reference's RNG consumption"
                                     if args.mode == "parity" else "fast: binary32 macro-cell DDA + ratio tracking"),
                       "tiles": "16x16 interleaved over ranks",
                       "l2": "flushed (256 MiB write) between timed frames",
                       "parallelism": f"tiles{world}", "gather": gather},
            "mrays_per_s": samples * world / (ms_per_step * 1e-3) / 1e6,
            "frame": frame_summary(stats, wall),
            "roofline": roofline_for(args.mode, stats, peaks, peak_kind, traffic),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "fast": fast,
            **extras,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def _sum_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def bench_extras(ctx, fc, params, peaks, rank=0, world=1, cam=None, rc=None, frame=None):
    """Part (c) photon-field queries/s and the config-3 KNN gather, aggregated
    over the ranks (each rank answers its own 2^22 / 2^20 query shard against
    the replicated field / photon map; weak scaling)."""
    import torch
    out = {}
    n = 1 << 22
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand((n, 3), device="cuda", generator=g)
    w = torch.rand((n, 2), device="cuda", generator=g)
    gg = torch.zeros(n, device="cuda")
    res = torch.empty((n, 3), device="cuda")
    for _ in range(3):
        ctx.field_query(x, w, gg, out=res)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        ctx.field_query(x, w, gg, out=res)
    b.record()
    torch.cuda.synchronize()
    dt = a.elapsed_time(b) / 5 / 1e3
    qps_rank = n / dt
    din = fc.pos.levels * fc.pos.features + fc.dir.levels * fc.dir.features + 1
    flop = 2 * (din * 64 + (fc.hidden_layers - 1) * 64 * 64 + 64 * 3)
    qps = _sum_over_ranks(qps_rank, world)
    gather = 2 * (fc.pos.levels * 8 * fc.pos.features + fc.dir.levels * 4 * fc.dir.features)
    hbm = float(peaks["hbm_gbs"]) * world
    tens = float(peaks["bf16_tflops"]) * world
    # random queries over the 170 MB paper tables: the hash-grid gathers (K3)
    # bound the query rate; the MLP (K4) is reported against the tensor peak
    out["field_query"] = {"queries_per_s": qps, "n_per_rank": n, "ranks": world, "scaling": "weak",
                          "flop_per_query": flop, "gather_bytes_per_query": gather,
                          "roofline": {"bound": "hbm", "kernel": "k_field_encode (dominant)",
                                       "achieved": qps * gather / 1e9, "peak": hbm, "unit": "GB/s",
                                       "frac": qps * gather / 1e9 / hbm,
                                       "per_unit": f"{gather} B (8 / 4 corners x F fp16 features x levels) per query"},
                          "roofline_mlp": {"bound": "tensor", "achieved": qps * flop / 1e12, "peak": tens,
                                           "unit": "TFLOP/s", "frac": qps * flop / 1e12 / tens}}
    # f1: photon tracing (Alg. 1) of 1M photons through this scene, binary64
    # (the paper's smallest map: 4.2-23.8 s on 2x Xeon)
    from paper_2304_07338_b200.api import TraceConfig
    tc = TraceConfig(n_total=1_000_000, seed=3)
    ctx.set_timing(True)
    for _ in range(2):
        tr = ctx.trace_photons(tc, device=True)
    ts = [], []
    for _ in range(3):
        tr = ctx.trace_photons(tc, device=True)
        st = ctx.trace_stats()
        ts[0].append(st["ms_trace"])
        ts[1].append(st["ms_compact"])
    ctx.set_timing(False)
    ms = float(np.median(ts[0])) + float(np.median(ts[1]))
    out["photon_trace"] = {"photons_per_s": _sum_over_ranks(tc.n_total / (ms / 1e3), world),
                           "n_photons": tc.n_total, "deposits": int(tr.photons.shape[0]),
                           "ms_trace": float(np.median(ts[0])), "ms_compact": float(np.median(ts[1])),
                           "tentative_collisions": st["tentative_collisions"], "precision": "f64",
                           "ranks": world, "scaling": "weak"}
    del tr
    sys.path.insert(0, str(ROOT / "tools"))
    if cam is not None:
        ctx.knn_build_traced(tc.phase_set)  # the 1M-photon map just traced
        out["renderers"] = bench_renderers(ctx, cam, rc, frame, world)
    # f2: paper-scale field training (2^16 queries / step, K = 1024 targets over
    # the traced map, paper field): make_batch vs train_step device time
    import bench_train
    out["field_training"] = bench_train.run(ctx, steps=10)
    out["field_training"]["ranks"] = world
    # config 3: KNN radiance estimate (k = 64) over 4M-photon 3-phase maps
    # (uniform, clustered, traced) x r_max in {inf, 0.05, 0.25}, 2^20
    # device-resident Stream::Train queries per batch, CUDA-event timed
    sys.path.insert(0, str(ROOT / "tools"))
    import bench_knn
    k = bench_knn.run(ctx, hbm_gbs=float(peaks["hbm_gbs"]))
    k["queries_per_s"] = _sum_over_ranks(k["queries_per_s"], world)
    k["algorithmic_GBps"] = _sum_over_ranks(k["algorithmic_GBps"], world)
    k["ranks"], k["scaling"] = world, "weak"
    hbm = float(peaks["hbm_gbs"]) * world
    k["roofline"] = {"bound": "hbm", "achieved": k["algorithmic_GBps"], "peak": hbm, "unit": "GB/s",
                     "frac": k["algorithmic_GBps"] / hbm, "per_unit": "2560 B (K=64 x 40-B records) per query"}
    out["knn_gather"] = k
    return out


def bench_renderers(ctx, cam, rc, frame, world=1):
    """The SPEC's comparison renderers on the headline frame (this rank's tiles):
    render_path_traced (16 vertices, NEE + HG continuation + roulette) -- the
    paper's path tracer of Table 2 -- and render_photon_map
    (K = 64 over the traced 1M-photon map), next to
    render_neural.  CUDA events on the render stream, mean of 3 frames."""
    import torch
    from paper_2304_07338_b200 import PathTraceConfig

    def timed(fn, n=3):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / n
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    neural = timed(lambda: ctx.render_neural(cam, rc, out=frame))
    pt = PathTraceConfig()
    path = timed(lambda: ctx.render_path_traced(cam, rc, pt, out=frame))
    pm = timed(lambda: ctx.render_photon_map(cam, rc, K=64, out=frame))
    return {"ms_neural": neural, "ms_path_traced": path, "ms_photon_map": pm,
            "speedup_neural_vs_path_traced": path / neural, "speedup_neural_vs_photon_map": pm / neural,
            "path_traced": {"max_bounces": pt.max_bounces, "rr_start_bounce": pt.rr_start_bounce},
            "photon_map": {"photons": "1M traced (Alg. 1), 3 phases", "K": 64, "r_max": "inf"},
            "mode": rc.mode, "note": "same frame, camera, seed and first interactions for all three"}


if __name__ == "__main__":
    sys.exit(main())
