#!/usr/bin/env python3
"""bench.py -- frames/s and per-stage ms of the per-frame pipeline on BASELINE.json's C2 workload
(synthetic tractography bundles, ~1 M segments, 256^3 grid, 1920x1080 opaque + cone-traced AO,
strategy vcsv), full rebuild every frame (upload + clip normals + grid refit -> voxelize -> mips ->
cull -> scan -> scatter/order -> shade -> trace).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload c1|c2|c3|c4]

One JSON line on stdout (rank 0).  `value` = whole-job frames/s with the f32 vertices already in
HBM; `e2e` = the same with pinned-host vertices copied in and the sRGB image + hit ids copied
out every step.  By default three frames of the dynamic sequence are in flight per GPU (three
engines on three streams, `--pipeline 3`): every frame runs the complete pipeline, the next
frame's build fills the issue slots this frame's latency-bound trace leaves free.  The per-stage
times, the roofline numbers and `config.serial_frames_per_s` come from a strictly serial pass
(`--pipeline 1` makes that the headline as well).  N > 1: every rank renders its own frames of a dynamic sequence (frame
sharding, no data-path collective; "weak").  `--impl reference` times the CPU oracle port
(the reference is Python+numba and cannot travel to the GPU box) on all host threads.
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (generator kwargs, res, width, height, strategy, mode, alpha)
    "c1": (dict(kind="random_streamlines", seed=0, polylines=100, verts_per_line=101), 64, 256, 256, "vcsv", "opaque", 1.0),
    "c2": (dict(kind="bundles", seed=0, n_bundles=40, fibers=250, verts=101), 256, 1920, 1080, "vcsv", "opaque", 1.0),
    "c3": (dict(kind="bundles", seed=0, n_bundles=40, fibers=250, verts=101), 256, 1920, 1080, "vsv", "transparent", 0.3),
    "c4": (dict(kind="bundles", seed=1, n_bundles=400, fibers=250, verts=101), 512, 1920, 1080, "vcsv", "opaque", 1.0),
    # unsteady-flow pathline sequence: every frame is a different time step (its own generator seed)
    "c5": (dict(kind="random_streamlines", seed=0, polylines=20000, verts_per_line=101, domain=128.0, curl=0.3),
           256, 1920, 1080, "vcsv", "opaque", 1.0),
}
C5_TIME_STEPS = 2      # distinct time steps generated on the host (~20 s each); the sequence cycles through them
R_VOXELS = 0.2
R_MIN = 0.5
LIGHT = "-0.5,-0.3,-0.8"


def describe(name, ls):
    gen, res, w, h, strat, mode, alpha = WORKLOADS[name]
    g = ",".join(f"{k}={v}" for k, v in gen.items() if k != "kind")
    return (f"{name.upper()}: {gen['kind']}({g}) = {ls.n_segments} segments / {ls.n_vertices} vertices, "
            f"{res}^3 grid, {w}x{h}, {mode}" + (f" alpha={alpha}" if mode == "transparent" else "")
            + f" + AO, strategy {strat}, r={R_VOXELS} voxel, full rebuild per frame")


def make_workload(name, bundle_fraction=1.0):
    import paper_2510_09081_b200 as lvx
    gen, res, w, h, strat, mode, alpha = WORKLOADS[name]
    gen = dict(gen)
    kind = gen.pop("kind")
    full = lvx.generate(kind, **gen)
    g, r_world = lvx.fit_grid(full, res, radius_voxels=R_VOXELS)
    ls = full
    if bundle_fraction < 1.0:
        keep = max(1, int(round(full.n_polylines * bundle_fraction)))
        end = int(full.polyline_offsets[keep])
        ls = lvx.LineSet(full.vertices[:end], full.polyline_offsets[:keep + 1], full.radius)
    cfg = lvx.PipelineConfig(res=res, width=w, height=h, strategy=strat, mode=mode, alpha=alpha, light=LIGHT)
    cam = lvx.make_camera(cfg, g)
    return full, ls, g, r_world, cam, cfg


def deform(verts, t, voxel_size):
    """C3's per-frame animation: y += 0.5*voxel*sin(2*pi*t/60 + 0.05*x)."""
    out = verts.copy()
    out[:, 1] += (0.5 * voxel_size * np.sin(2 * np.pi * t / 60.0 + 0.05 * verts[:, 0])).astype(np.float32)
    return out


class ClockSampler:
    """nvidia-smi clocks/throttle reasons during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(gpu_index)], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            pass

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.p is None:
            return out
        time.sleep(0.15)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            c = [x.strip() for x in line.split(",")]
            if len(c) < 9:
                continue
            try:
                sm.append(float(c[1])); mx.append(float(c[2]))
            except ValueError:
                continue
            for nm, val in zip(names, c[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.f.name)
        if sm:
            out.update(sm_mhz=float(np.median(sm)), sm_max_mhz=float(max(mx)), reasons=sorted(reasons), samples=len(sm))
        return out


def algorithmic_bytes(stats, n_verts, V, pixels):
    """compulsory streams + one 4-byte read-modify-write per atomic."""
    I, F, T, Vv = stats["voxels_visited"], stats["fragments"], stats["ray_capsule_tests"], stats["shaded_voxels"]
    return {
        "upload": 12 * n_verts + 48 * n_verts,              # f32 in, f64 voxel-unit verts + f64 normals out
        "voxelize": 12 * n_verts + 4 * V + 8 * I,
        "mips": 4 * V + (4.0 / 7.0) * V,
        "cull": 4 * V + V + V / 7.0,
        "scan": 9 * V,
        "scatter": 12 * n_verts + 8 * F + 4 * F + 8 * F,      # cursor atomics + write + ordering pass
        "shade": (32.0 / 7.0) * V + V + 8 * Vv,
        "trace": 20 * pixels + 28 * T,
    }


def run_gpu(args):
    import torch
    import torch.distributed as dist
    import paper_2510_09081_b200 as lvx
    from paper_2510_09081_b200.frame import STAGES

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the B200 path has no CPU fallback)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    full, ls, g, r_world, cam, cfg = make_workload(args.workload)
    _, res, w, h, strat, mode, alpha = WORKLOADS[args.workload]
    eng = lvx.FrameEngine(res, w, h, strategy=strat, mode=mode, alpha=alpha, light=cfg.light_vector())
    eng.set_topology(ls.polyline_offsets, ls.n_vertices)
    # a dynamic sequence: every step gets its own deformed vertex set (rank r renders frames r, r+world, ...)
    n_variants = 4
    if args.workload == "c5":   # time steps = independent line sets of the same topology
        n_variants = C5_TIME_STEPS
        gen = dict(WORKLOADS["c5"][0]); kind = gen.pop("kind"); gen.pop("seed")
        host = [torch.from_numpy(ls.vertices if rank + world * i == 0 else
                                 lvx.generate(kind, seed=rank + world * i, **gen).vertices).pin_memory()
                for i in range(n_variants)]
    else:
        host = [torch.from_numpy(deform(ls.vertices, rank + world * i, g.voxel_size)).pin_memory() for i in range(n_variants)]
    dev = [hv.cuda() for hv in host]
    out_srgb = torch.empty((h, w, 3), dtype=torch.uint8).pin_memory()
    out_hit = torch.empty((h, w), dtype=torch.int32).pin_memory()

    def refit(e):
        """a3 of the hot path, every frame: AABB of the new vertices on the device (24-byte read-back),
        fit_grid and the orbit camera on the host (lv/pipeline.py:68-87, 40-47)."""
        g_i, rw_i = e.fit(radius_voxels=R_VOXELS)
        return lvx.make_camera(cfg, g_i), g_i, rw_i

    def step_resident(i):
        eng.load_vertices(dev[i % n_variants])          # D2D: inputs are resident in HBM
        return eng.run(*refit(eng))

    def step_e2e(i):
        eng.load_vertices(host[i % n_variants])         # H2D from pinned memory
        r = eng.run(*refit(eng))
        out_srgb.copy_(eng.srgb, non_blocking=True)     # D2H result
        out_hit.copy_(eng.hit_id, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return r

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn):
        for i in range(args.warmup):
            fn(i)
        barrier()
        stage = {s: 0.0 for s in STAGES}
        stage["_trace_kernel"] = 0.0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        last = None
        for i in range(args.steps):
            last = fn(args.warmup + i)
            for s in STAGES:
                stage[s] += last.stage_ms[s]
            stage["_trace_kernel"] += last.trace_kernel_ms
        e1.record()
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, {s: v / args.steps for s, v in stage.items()}, last

    # Frames in flight.  depth 1: one frame after the other on one stream.  depth D > 1: D engines on D
    # streams, frame i on engine i mod D -- the next frame's build overlaps this frame's trace (every
    # frame still runs its full pipeline; the per-stage times below come from the depth-1 pass).
    depth = max(1, args.pipeline)
    engines, streams = [eng], [torch.cuda.current_stream()]
    for _ in range(depth - 1):
        e2 = lvx.FrameEngine(res, w, h, strategy=strat, mode=mode, alpha=alpha, light=cfg.light_vector())
        e2.set_topology(ls.polyline_offsets, ls.n_vertices)
        engines.append(e2)
        streams.append(torch.cuda.Stream())
    out_bufs = [(out_srgb, out_hit)] + [(torch.empty_like(out_srgb).pin_memory(), torch.empty_like(out_hit).pin_memory())
                                        for _ in range(depth - 1)]

    def timed_pipelined(e2e):
        src = host if e2e else dev
        n_total = args.warmup + args.steps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        main = torch.cuda.current_stream()
        inflight = [False] * depth
        for i in range(n_total + depth):
            k = i % depth
            with torch.cuda.stream(streams[k]):
                if inflight[k]:
                    engines[k].collect()
                    inflight[k] = False
                if i < n_total:
                    if i == args.warmup:            # the timed region starts when frame `warmup` is submitted
                        for s in streams:
                            s.synchronize()
                        barrier()
                        e0.record(main)
                        streams[k].wait_event(e0)
                    engines[k].load_vertices(src[i % n_variants])
                    engines[k].submit(*refit(engines[k]))
                    if e2e:
                        out_bufs[k][0].copy_(engines[k].srgb, non_blocking=True)
                        out_bufs[k][1].copy_(engines[k].hit_id, non_blocking=True)
                    inflight[k] = True
        for s in streams:
            main.wait_stream(s)
        e1.record(main)
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([ms], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        return ms

    sampler = ClockSampler(local) if rank == 0 else None
    ms, stage_ms, last = timed(step_resident)
    ms_serial = ms
    if depth > 1:
        ms = timed_pipelined(False)
    clocks = sampler.stop() if sampler else None
    if depth > 1:
        ms_e2e = timed_pipelined(True)
    else:
        ms_e2e, _, _ = timed(step_e2e)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_kind = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback 6650 GB/s (B200_PROFILING.md)"
    V, P = res ** 3, w * h
    ab = algorithmic_bytes(last.stats, ls.n_vertices, V, P)
    stage_roof = {s: {"ms": round(stage_ms[s], 4), "alg_mb": round(ab[s] / 1e6, 2),
                      "gbs": round(ab[s] / (stage_ms[s] * 1e-3) / 1e9, 1) if stage_ms[s] > 0 else None,
                      "frac": round(ab[s] / (stage_ms[s] * 1e-3) / 1e9 / peak, 4) if stage_ms[s] > 0 else None}
                  for s in STAGES}
    top = max(STAGES, key=lambda s: stage_ms[s])
    trace_kernel = "k_render_opaque_coop" if mode == "opaque" else "k_render_transparent_coop"
    kernel_of = {"upload": "k_upload", "voxelize": "k_voxelize", "mips": "k_mip1", "cull": "k_visibility",
                 "scan": "k_scan", "scatter": "k_scatter+k_order", "shade": "k_shade", "trace": trace_kernel}
    # the dominant kernel, timed alone with CUDA events on its stream (trace kernel: events 6->7)
    top_ms = stage_ms["_trace_kernel"] if top == "trace" else stage_ms[top]
    top_gbs = ab[top] / (top_ms * 1e-3) / 1e9
    traffic = None
    try:   # DRAM bytes per launch of that kernel from the committed `ncu --set full` capture
        traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[args.workload][kernel_of[top]]
    except Exception:
        pass
    fps = world * args.steps / (ms * 1e-3)
    fps_e2e = world * args.steps / (ms_e2e * 1e-3)
    line = {
        "metric": "frames/sec (voxelize+cull+build+shade+trace, full rebuild per frame) at 1920x1080",
        "value": round(fps, 3), "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": describe(args.workload, ls), "segments": ls.n_segments, "grid": res,
                   "image": [w, h], "multi_gpu": "frame-sharded dynamic sequence, no collective",
                   "frames_in_flight": depth, "serial_frames_per_s": round(world * args.steps / (ms_serial * 1e-3), 3),
                   "l2": "no explicit flush: each frame streams > L2 (126 MB) of grid/fragment data "
                         f"({round((sum(ab.values())) / 1e6)} MB algorithmic) between reuses"},
        "stages_ms": {s: round(v, 4) for s, v in stage_ms.items() if not s.startswith("_")},
        "frame_stats": {k: last.stats[k] for k in ("voxels_visited", "fragments", "occupied_voxels", "visible_voxels",
                                                   "solid_voxels", "ray_capsule_tests", "culled_fraction", "long_lists",
                                                   "wide_path", "shaded_voxels", "shading")},
        "e2e": {"value": round(fps_e2e, 3), "unit": "frames/s", "ms_per_step": round(ms_e2e / args.steps, 4),
                "h2d_bytes_per_step": int(host[0].numel() * 4),
                "d2h_bytes_per_step": int(out_srgb.numel() + out_hit.numel() * 4 + 128)},
        "gpu_launches": int((eng.kernel_launches_per_frame() + 3) * args.steps),   # + the 3 AABB kernels of the refit
        "roofline": {"bound": "hbm", "kernel": kernel_of[top], "stage": top,
                     "achieved": round(top_gbs, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(top_gbs / peak, 4), "traffic": traffic, "kernel_ms": round(top_ms, 4),
                     "algorithmic_bytes": int(ab[top]), "peak_source": peak_kind,
                     "per_stage": stage_roof},
        "clocks": clocks,
    }
    if not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args.workload, steps=1, warmup=0)
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(workload, steps, warmup, fraction=None):
    """The CPU oracle port (oracle/, C + OpenMP, all host threads) on a bounded sample of the
    workload: the first `fraction` of the bundles at the full grid/image; bundles are spatially
    separate, so every stage's work scales with the fraction and frames/s is scaled by it."""
    from oracle import oracle as orc
    orc.build()
    cores = orc.max_threads()
    _, res, w, h, strat, mode, alpha = WORKLOADS[workload]
    if fraction is None:
        fraction = 1.0
        if workload != "c1":
            # calibrate on 1/16 of the bundles, then take the largest sample that keeps the whole
            # run near `budget` seconds of CPU wall time
            budget = 25.0 if steps + warmup <= 1 else 150.0
            _, ls0, g0, rw0, cam0, cfg0 = make_workload(workload, 1.0 / 16)
            t0 = time.perf_counter()
            orc.run_frame(ls0, g0, rw0, cam0, cfg0.light_vector(), strategy=strat, mode=mode, alpha=alpha)
            est_full = 16.0 * (time.perf_counter() - t0)
            fraction = min(1.0, budget / ((steps + warmup) * est_full))
            fraction = max(fraction, 1.0 / 64)
    full, ls, g, r_world, cam, cfg = make_workload(workload, fraction)
    stage = {}
    times = []
    for i in range(warmup + steps):
        tm = {}
        t0 = time.perf_counter()
        orc.run_frame(ls, g, r_world, cam, cfg.light_vector(), strategy=strat, mode=mode, alpha=alpha, timings=tm)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
            for k, v in tm.items():
                stage[k] = stage.get(k, 0.0) + v / steps
    sec = float(np.mean(times))
    frac = ls.n_segments / full.n_segments
    return {"value": round(frac / sec, 5), "unit": "frames/s", "cores": cores, "kind": "port",
            "sample": f"{ls.n_segments} of {full.n_segments} segments (first {frac:.3f} of the polylines), full "
                      f"{res}^3 grid and {w}x{h} image; {sec:.2f} s per sample frame, value = fraction / seconds",
            "sample_seconds": round(sec, 3), "stages_ms_sample": {k: round(v, 1) for k, v in stage.items()}}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb = cpu_baseline(args.workload, steps=args.steps, warmup=args.warmup)
    full, ls, *_ = make_workload(args.workload)
    _, res, w, h, strat, mode, alpha = WORKLOADS[args.workload]
    line = {
        "impl": "reference",
        "metric": "frames/sec (voxelize+cull+build+shade+trace, full rebuild per frame) at 1920x1080",
        "value": cb["value"], "unit": "frames/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 / cb["value"], 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": describe(args.workload, ls), "segments": ls.n_segments, "grid": res, "image": [w, h]},
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--bundles", type=int, default=0, help="c2/c3/c4 only: number of fibre bundles (25 000 segments "
                                                           "each) instead of the workload's own, for segment-count sweeps")
    ap.add_argument("--pipeline", type=int, default=3, help="frames in flight per GPU (engines on separate streams); "
                                                             "1 = strictly one frame after the other")
    args = ap.parse_args()
    if args.bundles > 0:
        if WORKLOADS[args.workload][0]["kind"] != "bundles":
            ap.error("--bundles needs a bundles workload (c2, c3, c4)")
        WORKLOADS[args.workload][0]["n_bundles"] = args.bundles
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
