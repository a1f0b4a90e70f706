#!/bin/bash
# Full evidence round on the GPU box: parity tests, bench lines for every workload (+ reference arm), tiled
# emulation, ncu launch list and `--set full` captures.   usage (inside gpurun): bash tools/evidence_round.sh <tag>
TAG=${1:-rXX}
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/${TAG}_tests_gpu.log; cat $O/${TAG}_tests_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/${TAG}_bench_c2.json 2> $O/${TAG}_bench_c2.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/${TAG}_bench_c2_reference.json 2> $O/${TAG}_bench_c2_reference.err
timeout 600 python bench.py --steps 20 --warmup 3 --pipeline 1 --no-cpu --no-drop-in > $O/${TAG}_bench_c2_serial.json 2>> $O/${TAG}_bench_c2.err
for w in c3 c4 c1 c5 c2thick; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu > $O/${TAG}_bench_$w.json 2> $O/${TAG}_bench_$w.err
done
for a in 0.1 0.5; do
  timeout 600 python bench.py --workload c3 --alpha $a --steps 20 --warmup 3 --no-cpu --no-drop-in > $O/${TAG}_bench_c3_a$a.json 2> $O/${TAG}_bench_c3_a$a.err
done
timeout 600 python bench.py --workload c2 --bundles 160 --steps 10 --warmup 3 --no-cpu --no-drop-in > $O/${TAG}_bench_c2_4M.json 2> $O/${TAG}_bench_c2_4M.err
for G in 2 4 8; do
  timeout 600 python bench.py --workload c4 --emulate-world $G --steps 5 --warmup 3 --no-cpu > $O/${TAG}_emu_c4_g$G.json 2> $O/${TAG}_emu_c4_g$G.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/${TAG}_launches_c2.csv \
   python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu --no-drop-in --pipeline 1 > $O/${TAG}_launches_c2.log 2>&1
python tools/launch_summary.py $O/${TAG}_launches_c2.csv > $O/${TAG}_launches_c2_summary.txt 2>&1
for w in c2 c3 c4 c2thick; do
  # every kernel of one frame, summarised here (the report itself is too large to ship back)
  timeout 1200 ncu --set full --clock-control none \
     -k regex:'k_render|k_scatter|k_order$|k_voxelize|k_shade$|k_visibility|k_march|k_upload|k_pack_mip1|k_mip_next|k_solid|k_dilate|k_scan|k_resolve|k_nzmask|k_march_levels|k_need_list|k_ormip$|k_brick_flags|k_super_flags|k_superbrick_shadow' \
     --launch-skip ${NCU_SKIP:-66} -c 32 -o $O/${TAG}_all_$w -f python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --no-drop-in --pipeline 1 > $O/${TAG}_ncu_$w.log 2>&1
  python tools/ncu_summary.py $O/${TAG}_all_$w.ncu-rep $O/ncu_traffic.json $w > $O/${TAG}_ncu_full_${w}_summary.txt 2>&1
  rm -f $O/${TAG}_all_$w.ncu-rep
done
for w in c2 c3; do
  # the trace kernel with source-level counters
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_render' --launch-skip 3 -c 1 \
     -o $O/${TAG}_trace_$w -f python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --no-drop-in --pipeline 1 >> $O/${TAG}_ncu_$w.log 2>&1
  python tools/ncu_lines.py $O/${TAG}_trace_$w.ncu-rep 40 > $O/${TAG}_ncu_trace_${w}_lines.txt 2>&1
  rm -f $O/${TAG}_trace_$w.ncu-rep
done
for f in $O/${TAG}_bench_*.json $O/${TAG}_emu_*.json; do python - $f <<'P'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1].split("/")[-1], d.get("value"), d.get("unit"), "serial", d.get("run", {}).get("serial_frames_per_s"),
          "e2e", d.get("e2e", {}).get("value"), d.get("stages_ms"), "drop_in", d.get("drop_in", {}).get("frames_per_s"),
          "cpu", d.get("cpu_baseline", {}).get("value"))
except Exception as e:
    print(sys.argv[1], "FAILED", e)
P
done
