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
times, the roofline numbers and `run.serial_frames_per_s` come from a strictly serial pass
(`--pipeline 1` makes that the headline as well).

N > 1 (`--gpus N`: under torchrun WORLD_SIZE must equal N; without torchrun the script spawns the N ranks
itself): `--multi frames` (default) -- every rank renders its own frames of a dynamic sequence (frame
sharding, no data-path collective; "weak"); `--multi tiled` -- all ranks render EVERY frame together
(TiledFrame: segment-sharded voxelization, NCCL all-reduce of the 64-bit occupancy accumulators,
tile-restricted build, per-rank screen tile, gather on rank 0; "strong").  `--emulate-world G` plays the G
ranks of a tiled job one after the other on ONE GPU (no exchange) and prints their per-rank stage times.

`--impl reference` times the CPU oracle port (the reference is Python+numba and cannot travel to the
GPU box) on all host threads: the whole workload for C1/C2/C3/C5, a stated sample for C4.
"""
import argparse
import glob
import hashlib
import json
import os
import socket
import subprocess
import sys
import tempfile
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
# culling-active variant of C2: the same bundles drawn as thick tubes (radius 0.6 voxel), so that bundle
# interiors become solid (eroded occupancy >= 0.999) and the voxels behind them are culled
WORKLOADS["c2thick"] = WORKLOADS["c2"]
C5_TIME_STEPS = 100    # the sequence has 100 time steps (seed = time step); a run generates the ones it renders (~0.5 s each)
R_VOXELS = 0.2
R_VOXELS_OF = {"c2thick": 0.6}
R_MIN = 0.5
LIGHT = "-0.5,-0.3,-0.8"


def radius_of(name):
    return R_VOXELS_OF.get(name, R_VOXELS)


def describe(name, ls):
    gen, res, w, h, strat, mode, alpha = WORKLOADS[name]
    g = ",".join(f"{k}={v}" for k, v in gen.items() if k != "kind")
    return (f"{name.upper()}: {gen['kind']}({g}) = {ls.n_segments} segments / {ls.n_vertices} vertices, "
            f"{res}^3 grid, {w}x{h}, {mode}" + (f" alpha={alpha}" if mode == "transparent" else "")
            + f" + AO, strategy {strat}, r={radius_of(name)} voxel, full rebuild per frame")


def workload_config(name, ls):
    """`config` of the JSON line: names the workload only, identical in the GPU and the reference arm."""
    _, res, w, h, *_ = WORKLOADS[name]
    l2 = ("no explicit flush: every frame streams more than L2 (126 MB) of grid and fragment data between reuses"
          if res >= 256 else "no flush; this small parity config fits in L2 and is not a bench line")
    return {"workload": describe(name, ls), "segments": ls.n_segments, "grid": res, "image": [w, h], "l2": l2}


def csrc_sha16():
    hsh = hashlib.sha256()
    for f in sorted(glob.glob(os.path.join(ROOT, "paper_2510_09081_b200", "csrc", "*.cu*"))):
        hsh.update(open(f, "rb").read())
    return hsh.hexdigest()[:16]


def make_workload(name, bundle_fraction=1.0):
    import paper_2510_09081_b200 as lvx
    gen, res, w, h, strat, mode, alpha = WORKLOADS[name]
    gen = dict(gen)
    kind = gen.pop("kind")
    full = lvx.generate(kind, **gen)
    g, r_world = lvx.fit_grid(full, res, radius_voxels=radius_of(name))
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


def load_traffic(workload, kernel):
    """DRAM bytes per launch of `kernel` from the committed `ncu --set full` capture (profiles/ncu_traffic.json,
    written by tools/ncu_summary.py together with the hash of csrc/ it was taken on).  A capture of other
    kernel sources is refused: (None, why)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        j = json.load(open(path))
        names = kernel.split("+")
        val = sum(int(j[workload][k]) for k in names)
    except Exception as e:
        return None, f"no capture for {workload}/{kernel} in profiles/ncu_traffic.json ({type(e).__name__})"
    have, now = (j.get("_csrc_sha16") or {}).get(workload), csrc_sha16()
    if have != now:
        return None, f"stale: profiles/ncu_traffic.json[{workload}] was captured on csrc {have}, this build is {now}"
    return val, f"profiles/ncu_traffic.json (ncu --set full, dram read+write of one launch, csrc {now})"


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
    rv = radius_of(args.workload)
    if args.multi == "tiled" or args.emulate_world > 1:
        return run_tiled(args, lvx, torch, dist, rank, world, local, ls, g, cfg)
    eng = lvx.FrameEngine(res, w, h, strategy=strat, mode=mode, alpha=alpha, light=cfg.light_vector())
    eng.set_topology(ls.polyline_offsets, ls.n_vertices)
    # a dynamic sequence: every step gets its own deformed vertex set (rank r renders frames r, r+world, ...)
    n_variants = 4
    if args.workload == "c5":   # time steps = independent line sets of the same topology
        n_variants = min(C5_TIME_STEPS, args.warmup + args.steps)     # frame i of this rank = time step rank + world * i
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
        g_i, rw_i = e.fit(radius_voxels=rv)
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
    drop_in = None
    if world == 1 and not args.no_drop_in:
        drop_in = time_drop_in(args, lvx, torch, ls, host, out_srgb, out_hit, n_variants, rv)
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
    traffic, traffic_source = load_traffic(args.workload, kernel_of[top])
    fps = world * args.steps / (ms * 1e-3)
    fps_e2e = world * args.steps / (ms_e2e * 1e-3)
    line = {
        "metric": "frames/sec (voxelize+cull+build+shade+trace, full rebuild per frame) at 1920x1080",
        "value": round(fps, 3), "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload, ls),
        "run": {"multi_gpu": "frame-sharded dynamic sequence, no collective", "frames_in_flight": depth,
                "serial_frames_per_s": round(world * args.steps / (ms_serial * 1e-3), 3),
                "serial_ms_per_step": round(ms_serial / args.steps, 4),
                "algorithmic_mb_per_frame": round(sum(ab.values()) / 1e6)},
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
                     "frac": round(top_gbs / peak, 4), "traffic": traffic, "traffic_source": traffic_source,
                     "kernel_ms": round(top_ms, 4),
                     "algorithmic_bytes": int(ab[top]), "peak_source": peak_kind,
                     "per_stage": stage_roof},
        "clocks": clocks,
    }
    if os.environ.get("LVX_DEBUG_STATS"):
        line["raw_stats"] = last.raw_stats
    if drop_in is not None:
        line["drop_in"] = drop_in
    if not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args.workload, steps=1, warmup=0)
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def time_drop_in(args, lvx, torch, ls, host, out_srgb, out_hit, n_variants, rv):
    """The same frames through the reference-shaped entry point (lv/pipeline.py:50-150): `ScenePipeline`
    with cfg.revoxelize, new vertices per frame via update_vertices (pinned host -> HBM), render_frame()
    returning an Image that owns its pixels, sRGB + hit ids copied back.  Two host synchronisations and
    fresh output tensors per frame -- the price of the reference's stage-by-stage contract."""
    _, res, w, h, strat, mode, alpha = WORKLOADS[args.workload]
    cfg = lvx.PipelineConfig(res=res, width=w, height=h, strategy=strat, mode=mode, alpha=alpha, light=LIGHT,
                             r=rv, revoxelize=True)
    pipe = lvx.ScenePipeline(cfg, lineset_override=ls)

    def frame(i):
        pipe.update_vertices(host[i % n_variants])
        img = pipe.render_frame()
        out_srgb.copy_(img.srgb_dev, non_blocking=True)
        out_hit.copy_(img.hit_id_dev, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    for i in range(args.warmup):
        frame(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        frame(args.warmup + i)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return {"api": "ScenePipeline(cfg.revoxelize).update_vertices(pinned host) + render_frame() -> Image, "
                   "sRGB + hit ids copied to the host", "frames_per_s": round(args.steps / (ms * 1e-3), 3),
            "ms_per_step": round(ms / args.steps, 4)}


def run_tiled(args, lvx, torch, dist, rank, world, local, ls, g, cfg):
    """All ranks render every frame together (SURVEY.md §8e 1+2, C4's multi-GPU mode): rank r voxelizes its
    segment shard, the 64-bit accumulators are all-reduced (NCCL), every rank culls on the merged grid, builds
    the A-buffer and the shading for the voxels of its own screen strip and traces it; rank 0 gathers the
    strips.  `--emulate-world G` (one process, one GPU) plays the G ranks in turn without the exchange."""
    from paper_2510_09081_b200 import distributed as D
    from paper_2510_09081_b200.frame import STAGES
    _, res, w, h, strat, mode, alpha = WORKLOADS[args.workload]
    rv = radius_of(args.workload)
    emu = args.emulate_world if args.emulate_world > 1 else 0
    if emu and world > 1:
        raise SystemExit("bench.py: --emulate-world runs in one process on one GPU")
    eng = lvx.FrameEngine(res, w, h, strategy=strat, mode=mode, alpha=alpha, light=cfg.light_vector())
    eng.set_topology(ls.polyline_offsets, ls.n_vertices)
    n_variants = 4          # every rank holds the same deformed vertex sets: all ranks work on the same frame
    host = [torch.from_numpy(deform(ls.vertices, i, g.voxel_size)).pin_memory() for i in range(n_variants)]
    dev = [hv.cuda() for hv in host]
    out_srgb = torch.empty((h, w, 3), dtype=torch.uint8).pin_memory()
    out_hit = torch.empty((h, w), dtype=torch.int32).pin_memory()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def strip_work(stage):       # the part of a rank's frame that depends on its strip
        return sum(stage.get(k, 0.0) for k in ("scan", "scatter", "shade", "trace"))

    def frame(tf, i, e2e):
        eng.load_vertices((host if e2e else dev)[i % n_variants])
        g_i, rw_i = eng.fit(radius_voxels=rv)
        r = tf.run(lvx.make_camera(cfg, g_i), g_i, rw_i)
        srgb, hit = tf.gather_image()
        if e2e and srgb is not None:
            out_srgb[:srgb.shape[0]].copy_(srgb, non_blocking=True)
            out_hit[:hit.shape[0]].copy_(hit, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        return r

    def timed(tf, e2e):
        for i in range(args.warmup):
            r = frame(tf, i, e2e)
            if world > 1 and not e2e:         # strips follow the measured work of the warm-up frames, then stay put
                tf.rebalance(strip_work(r.stage_ms))
        barrier()
        stage, last = {}, None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.steps):
            last = frame(tf, args.warmup + i, e2e)
            for k, v in last.stage_ms.items():
                stage[k] = stage.get(k, 0.0) + v / args.steps
        e1.record()
        barrier()
        return e0.elapsed_time(e1), stage, last

    keys = ("fragments", "owned_voxels", "visible_voxels", "ray_capsule_tests", "voxels_visited", "shaded_voxels")
    sampler = ClockSampler(local) if rank == 0 else None
    if emu:
        def one_pass(rows):
            per_rank = []
            for r in range(emu):
                tf = D.TiledFrame(eng, comm=D.EmulatedComm(r, emu))
                if rows is not None:
                    tf.set_rows(rows)
                ms, stage, last = timed(tf, False)
                own = sum(v for k, v in stage.items() if k != "emulated_peers")
                per_rank.append({"rank": r, "tile": list(tf.tiles[r]), "segments": list(tf.seg_range()),
                                 "own_stage_ms_sum": round(own, 4), "strip_work_ms": round(strip_work(stage), 4),
                                 "stages_ms": {k: round(v, 4) for k, v in stage.items()},
                                 "stats": {k: last.stats[k] for k in keys}})
            return per_rank
        equal = one_pass(None)
        rows0 = [p["tile"][1] for p in equal] + [h]
        # strip balancing: what TiledFrame.rebalance does with the all-gathered numbers of the real job
        rows1 = D.balanced_rows(rows0, [p["strip_work_ms"] for p in equal], h)
        balanced = one_pass(rows1)
        clocks = sampler.stop()
        worst_eq = max(p["own_stage_ms_sum"] for p in equal)
        worst = max(p["own_stage_ms_sum"] for p in balanced)
        line = {
            "metric": "frames/sec (voxelize+cull+build+shade+trace, full rebuild per frame) at 1920x1080",
            "value": round(1e3 / worst, 3), "unit": "frames/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(worst, 4), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": workload_config(args.workload, ls),
            "emulated": {"world": emu, "note": "ONE GPU plays the ranks of a tiled job in turn; value = 1 / (largest per-rank "
                         "sum of the rank's own stage times) with strips balanced from the strip-dependent stage times "
                         "of a first pass on equal strips; the all-reduce of the accumulators (exchange_bytes per rank) "
                         "and the gather of the strips are NOT included", "exchange_bytes": 8 * res ** 3,
                         "equal_strips": {"rows": rows0, "slowest_rank_ms": round(worst_eq, 4), "ranks": equal},
                         "balanced_strips": {"rows": rows1, "slowest_rank_ms": round(worst, 4), "ranks": balanced},
                         "ranks": balanced},
            "gpu_launches": int((eng.kernel_launches_per_frame() + 3) * args.steps * emu * 2), "clocks": clocks}
        print(json.dumps(line))
        return

    tf = D.TiledFrame(eng)
    ms, stage, last = timed(tf, False)
    clocks = sampler.stop() if sampler else None
    ms_e2e, _, _ = timed(tf, True)
    t = torch.tensor([ms, ms_e2e], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, ms_e2e = (float(x) for x in t.tolist())
    mine = {"rank": rank, "tile": list(tf.tiles[rank]), "segments": list(tf.seg_range()),
            "stages_ms": {k: round(v, 4) for k, v in stage.items()}, "stats": {k: last.stats[k] for k in keys}}
    ranks = [mine]
    if world > 1:
        ranks = [None] * world
        dist.all_gather_object(ranks, mine)
    if rank == 0:
        xb = tf.exchange_bytes if world > 1 else 0
        xms = max((p["stages_ms"].get("exchange", 0.0) for p in ranks), default=0.0)
        line = {
            "metric": "frames/sec (voxelize+cull+build+shade+trace, full rebuild per frame) at 1920x1080",
            "value": round(args.steps / (ms * 1e-3), 3), "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.workload, ls),
            "run": {"multi_gpu": "tiled: segment-sharded voxelize + all-reduce of the occupancy grid (packed words or 64-bit accumulators) + per-rank "
                                 "screen strip (tile-restricted build) + gather on rank 0", "frames_in_flight": 1},
            "exchange": {"all_reduce_bytes_per_rank": xb, "kind": tf.exchange_kind if world > 1 else None,
                         "note": "packed = 4-byte words after a 16-byte pre-check (no field of the merged grid can overflow), "
                                 "wide = the 8-byte accumulators; all_reduce_ms includes the pre-check and the pack pass",
                         "all_reduce_ms_max": round(xms, 4),
                         "bus_gbs": round(2 * (world - 1) / world * xb / (xms * 1e-3) / 1e9, 1) if xms > 0 else None,
                         "gather_bytes": int(out_srgb.numel() + out_hit.numel() * 4)},
            "ranks": ranks,
            "e2e": {"value": round(args.steps / (ms_e2e * 1e-3), 3), "unit": "frames/s",
                    "ms_per_step": round(ms_e2e / args.steps, 4),
                    "h2d_bytes_per_step": int(host[0].numel() * 4) * world,
                    "d2h_bytes_per_step": int(out_srgb.numel() + out_hit.numel() * 4 + 128 * world)},
            "gpu_launches": int((eng.kernel_launches_per_frame() + 3) * args.steps * world), "clocks": clocks}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(workload, steps, warmup, fraction=None):
    """The CPU oracle port (oracle/, C + OpenMP, all host threads).  C1/C2/C3/C5: the WHOLE workload, every
    step one full frame, value = 1 / measured seconds per frame.  C4 (10 M segments at 512^3 needs tens of
    seconds and tens of GB per frame on the host): a stated sample -- the first 1/8 of the bundles at the full
    grid and image; bundles are spatially separate, so the build work scales with the fraction while the
    per-voxel / per-pixel sweeps do not, and value = fraction / seconds is an upper bound for the CPU."""
    from oracle import oracle as orc
    orc.build()
    orc.set_threads(len(os.sched_getaffinity(0)))     # all host threads (torchrun exports OMP_NUM_THREADS=1)
    cores = orc.max_threads()
    _, res, w, h, strat, mode, alpha = WORKLOADS[workload]
    if fraction is None:
        fraction = 0.125 if workload == "c4" else 1.0
    full, ls, g, r_world, cam, cfg = make_workload(workload, fraction)
    stage = {}
    times = []
    for i in range(warmup + steps):
        tm = {}
        # a dynamic sequence like the GPU arm's: every step has its own deformed vertex set
        ls_i = type(ls)(deform(ls.vertices, i, g.voxel_size), ls.polyline_offsets, ls.radius) if workload != "c5" else ls
        t0 = time.perf_counter()
        orc.run_frame(ls_i, g, r_world, cam, cfg.light_vector(), strategy=strat, mode=mode, alpha=alpha, timings=tm)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
            for k, v in tm.items():
                stage[k] = stage.get(k, 0.0) + v / steps
    sec = float(np.mean(times))
    frac = ls.n_segments / full.n_segments
    whole = ls.n_segments == full.n_segments
    sample = (f"the whole workload: {ls.n_segments} segments, {res}^3 grid, {w}x{h} image; {len(times)} frame(s) of "
              f"{sec:.2f} s each, value = 1 / seconds per frame" if whole else
              f"{ls.n_segments} of {full.n_segments} segments (first {frac:.3f} of the polylines), full "
              f"{res}^3 grid and {w}x{h} image; {sec:.2f} s per sample frame, value = fraction / seconds")
    return {"value": round(frac / sec, 5), "unit": "frames/s", "cores": cores, "kind": "port",
            "sample": sample, "whole_workload": whole, "sample_seconds": round(sec, 3),
            "total_seconds": round(float(np.sum(times)), 2),
            "stages_ms_sample": {k: round(v, 1) for k, v in stage.items()}}


def reference_package_probe():
    """Whether the reference's own package can run on this host: it needs numba, and its pip-installed copy
    under baseline/_ref (git-ignored; `python -m pip install --no-index --no-build-isolation --no-deps --target
    baseline/_ref <copy of /root/reference/pkg>`, done by __graft_entry__.build() where /root/reference exists)."""
    out = {}
    try:
        import numba
        out["numba"] = numba.__version__
    except Exception as e:
        out["numba"] = f"not importable ({type(e).__name__})"
    out["baseline_ref_present"] = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "linevox"))
    return out


def time_reference_package(workload):
    """ONE frame of the workload through the UNMODIFIED reference package (linevox: Python + numba, all host
    threads) and its own entry point: the line set is written as a .lns file with the reference's writer,
    `linevox.ScenePipeline(PipelineConfig(input=<file>, ...))` loads, voxelizes, culls, builds, shades and
    renders it.  frames/s = 1 / (sum of the reference's own five stage timers), its definition of the frame
    (lv/pipeline.py:68-136; file loading and the per-polyline Python loop of compute_clip_normals are its
    `load_ms`, reported beside).  JIT compilation happens before, on a tiny scene of the same mode."""
    info = reference_package_probe()
    if not info["baseline_ref_present"] or "not importable" in info["numba"] or workload == "c4":
        info["ran"] = False
        if workload == "c4":
            info["why"] = "C4 (512^3, 10 M segments) needs tens of GB and minutes per frame in the reference"
        return info
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "lvx_numba_cache"))
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    try:
        import linevox as lv
        import numba
        numba.set_num_threads(min(numba.config.NUMBA_NUM_THREADS, len(os.sched_getaffinity(0))))
        threads = numba.get_num_threads()
        _, res, w, h, strat, mode, alpha = WORKLOADS[workload]
        full, ls, *_ = make_workload(workload)
        t0 = time.perf_counter()
        lv.ScenePipeline(lv.PipelineConfig(input="gen:helix?turns=2&verts=60", res=32, width=32, height=32,
                                           strategy=strat, mode=mode, alpha=alpha, light=LIGHT)).render_frame()
        jit_s = time.perf_counter() - t0
        path = os.path.join(tempfile.gettempdir(), f"lvx_{workload}.lns")
        lv.save_lineset(lv.LineSet(ls.vertices, ls.polyline_offsets, ls.radius), path)
        cfg = lv.PipelineConfig(input=path, res=res, width=w, height=h, strategy=strat, mode=mode, alpha=alpha,
                                light=LIGHT, r=radius_of(workload))
        t0 = time.perf_counter()
        pipe = lv.ScenePipeline(cfg)          # build_geometry: load + clip normals + fit + voxelize
        img = pipe.render_frame()
        wall = time.perf_counter() - t0
        os.unlink(path)
        st = pipe.stats
        stages = {k: round(float(st[k]), 1) for k in ("voxelize_ms", "cull_ms", "abuffer_ms", "shading_ms", "render_ms")}
        frame_s = sum(stages.values()) * 1e-3
        info.update(ran=True, kind="reference", threads=threads, jit_warmup_s=round(jit_s, 1),
                    frames_per_s=round(1.0 / frame_s, 5), frame_seconds=round(frame_s, 2),
                    wall_seconds_incl_load=round(wall, 2), load_ms=round(float(st["load_ms"]), 1),
                    stages_ms=stages, fragments=int(st["fragments"]), ray_capsule_tests=int(st["ray_capsule_tests"]),
                    hits=int((img.hit_id >= 0).sum()))
    except Exception as e:          # the reference arm must still print its line
        info.update(ran=False, why=f"{type(e).__name__}: {e}"[:300])
    return info


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb = cpu_baseline(args.workload, steps=args.steps, warmup=args.warmup)
    full, ls, *_ = make_workload(args.workload)
    ms_step = 1e3 * cb["sample_seconds"] if cb["whole_workload"] else 1e3 / cb["value"]
    line = {
        "impl": "reference",
        "metric": "frames/sec (voxelize+cull+build+shade+trace, full rebuild per frame) at 1920x1080",
        "value": cb["value"], "unit": "frames/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload, ls),
        "cpu_baseline": cb,
        "reference_package": (reference_package_probe() if args.no_ref_package else time_reference_package(args.workload)),
        "e2e": {"value": cb["value"], "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))


def free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(n):
    """`bench.py --gpus N` outside torchrun: start the N ranks exactly as the driver would."""
    if "--impl" not in sys.argv or "reference" not in sys.argv:
        import torch
        have = torch.cuda.device_count()
        if have < n:
            raise SystemExit(f"bench.py: --gpus {n} but this host has {have} CUDA device(s)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-ref-package", action="store_true", help="--impl reference: do not time the real reference "
                                                                   "package (baseline/_ref) beside the C port")
    ap.add_argument("--no-drop-in", action="store_true", help="skip the ScenePipeline (reference-shaped API) timing")
    ap.add_argument("--bundles", type=int, default=0, help="c2/c3/c4 only: number of fibre bundles (25 000 segments "
                                                           "each) instead of the workload's own, for segment-count sweeps")
    ap.add_argument("--pipeline", type=int, default=3, help="frames in flight per GPU (engines on separate streams); "
                                                             "1 = strictly one frame after the other")
    ap.add_argument("--multi", default="frames", choices=["frames", "tiled"],
                    help="N > 1: frames = every rank renders its own frames (weak); tiled = all ranks render every "
                         "frame together: sharded voxelize + all-reduce + screen strips (strong)")
    ap.add_argument("--emulate-world", type=int, default=0, help="one GPU plays the G ranks of a tiled job in turn")
    ap.add_argument("--alpha", type=float, default=None, help="opacity of a transparent workload (c3: 0.1 .. 0.5)")
    args = ap.parse_args()
    env_world = os.environ.get("WORLD_SIZE")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if env_world is None and args.gpus > 1:
        spawn_ranks(args.gpus)
    if env_world is not None and int(env_world) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started WORLD_SIZE={env_world} ranks; "
                         "pass --gpus equal to the number of ranks")
    if args.alpha is not None:
        wl = WORKLOADS[args.workload]
        if wl[5] != "transparent" or not 0.0 < args.alpha <= 1.0:
            ap.error("--alpha needs a transparent workload (c3) and a value in (0, 1]")
        WORKLOADS[args.workload] = wl[:6] + (args.alpha,)
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
