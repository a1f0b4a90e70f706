#!/bin/bash
# BASELINE.json's metric: frames/s and per-stage ms at 1080p vs segment count.  usage (inside gpurun): bash tools/sweep.sh <tag>
TAG=${1:-rXX}; O=gpurun_out; mkdir -p $O
for w in c2 c3; do
  : > $O/${TAG}_sweep_segments_$w.jsonl
  for n in 1 4 12 40 80 160; do
    [ $w = c3 ] && [ $n = 160 ] && continue
    timeout 600 python bench.py --workload $w --bundles $n --steps 20 --warmup 3 --no-cpu --no-drop-in 2>/dev/null >> $O/${TAG}_sweep_segments_$w.jsonl
  done
done
python - $O/${TAG}_sweep_segments_c2.jsonl $O/${TAG}_sweep_segments_c3.jsonl <<'P'
import json, sys
print("| workload | segments | frames/s (3 in flight) | serial | e2e | voxelize | cull | scatter | shade | trace (ms) |")
print("|---|---|---|---|---|---|---|---|---|---|")
for f in sys.argv[1:]:
    for line in open(f):
        line = line.strip()
        if not line: continue
        d = json.loads(line); s = d["stages_ms"]
        print(f"| {d['config']['workload'][:2]} | {d['config']['segments']:,} | {d['value']:.1f} | {d['run']['serial_frames_per_s']:.1f} | {d['e2e']['value']:.1f} | "
              f"{s['voxelize']:.2f} | {s['cull']:.2f} | {s['scan'] + s['scatter']:.2f} | {s['shade']:.2f} | {s['trace']:.2f} |".replace(",", " "))
P
