#!/bin/bash
# Full evidence round on the GPU box: parity tests, bench lines for every workload (+ reference arm),
# ncu launch list and `--set full` captures.   usage (inside gpurun): bash tools/evidence_round.sh <tag>
TAG=${1:-rXX}
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/${TAG}_tests_gpu.log; cat $O/${TAG}_tests_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 > $O/${TAG}_bench_c2.json 2> $O/${TAG}_bench_c2.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/${TAG}_bench_c2_reference.json 2> $O/${TAG}_bench_c2_reference.err
timeout 600 python bench.py --steps 20 --warmup 3 --pipeline 1 --no-cpu > $O/${TAG}_bench_c2_serial.json 2>> $O/${TAG}_bench_c2.err
for w in c3 c4 c1 c5; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu > $O/${TAG}_bench_$w.json 2> $O/${TAG}_bench_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/${TAG}_launches_c2.csv \
   python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu --pipeline 1 > $O/${TAG}_launches_c2.log 2>&1
for w in c2 c3; do
  # every kernel of one frame, summarised here (the report itself is too large to ship back)
  timeout 900 ncu --set full --clock-control none \
     -k regex:'k_render|k_scatter|k_order|k_voxelize|k_shade$|k_visibility|k_march$|k_upload|k_mip1|k_solid|k_dilate|k_scan|k_resolve|k_nzmask|k_init_cursor|k_march_levels' \
     --launch-skip ${NCU_SKIP:-60} -c 24 -o $O/${TAG}_all_$w -f python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --pipeline 1 > $O/${TAG}_ncu_$w.log 2>&1
  python tools/ncu_summary.py $O/${TAG}_all_$w.ncu-rep $O/${TAG}_ncu_traffic.json $w > $O/${TAG}_ncu_full_${w}_summary.txt 2>&1
  rm -f $O/${TAG}_all_$w.ncu-rep
  # the trace kernel with source-level counters
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_render' --launch-skip 3 -c 1 \
     -o $O/${TAG}_trace_$w -f python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --pipeline 1 >> $O/${TAG}_ncu_$w.log 2>&1
done
for f in $O/${TAG}_bench_*.json; do python - $f <<'P'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1].split("/")[-1], d.get("value"), d.get("unit"), "serial", d.get("config", {}).get("serial_frames_per_s"),
          "e2e", d.get("e2e", {}).get("value"), d.get("stages_ms"), "cpu", d.get("cpu_baseline", {}).get("value"))
except Exception as e:
    print(sys.argv[1], "FAILED", e)
P
done
