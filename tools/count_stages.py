#!/usr/bin/env python3
"""Debug: run one frame of a bench workload with a -DLVX_COUNT build and print the per-stage work
counters of the trace kernel (stats words 12..15).  usage: LVX_LIB=.../liblvx_b200_cnt.so tools/count_stages.py c3"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, torch
import paper_2510_09081_b200 as lvx
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
full, ls, g, r_world, cam, cfg = bench.make_workload(name)
_, res, w, h, strat, mode, alpha = bench.WORKLOADS[name]
eng = lvx.FrameEngine(res, w, h, strategy=strat, mode=mode, alpha=alpha, light=cfg.light_vector())
eng.set_topology(ls.polyline_offsets, ls.n_vertices)
eng.load_vertices(torch.from_numpy(ls.vertices).cuda())
out = eng.run(cam, g, r_world)
st = eng.stats.cpu().numpy()
print(name, "ref tests", out.stats["ray_capsule_tests"], "fragments", out.stats["fragments"])
print("  LVX_COUNT=1: tight pairs", st[13], "f64 tests", st[14], "hits", st[15])
print("  LVX_COUNT=2: rounds", st[13], "active lanes", st[14], "march iterations", st[15], "marching lanes", st[11])
print("  stage ms", out.stage_ms)
