#!/bin/bash
# quick GPU check: parity tests (-x) then serial bench lines.  usage: bash tools/quick.sh <tag> "<workloads>" [env...]
TAG=$1; WL=${2:-"c2 c4"}; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -6 > $O/${TAG}_tests_gpu.log; cat $O/${TAG}_tests_gpu.log
for w in $WL; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu > $O/${TAG}_bench_$w.json 2> $O/${TAG}_bench_$w.err
  python - $O/${TAG}_bench_$w.json $w <<'P'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], d["value"], "fps serial", d["run"]["serial_frames_per_s"], "e2e", d["e2e"]["value"], d["stages_ms"])
except Exception as e:
    print(sys.argv[2], "FAILED", e); print(open(sys.argv[1].replace(".json",".err")).read()[-2000:])
P
done
