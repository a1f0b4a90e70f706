#!/bin/bash
# One GPU-box round: parity tests, bench lines, ncu launch list + full capture of the hot kernels.
# usage (inside gpurun): [VARIANTS="b1 b2"] [NO_NCU=1] bash tools/gpu_round.sh <tag> [workloads...]
TAG=${1:-rXX}; shift
WL=${@:-c2 c3}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/tests_$TAG.log
cat gpurun_out/tests_$TAG.log
show() {
  python - "$1" "$2" <<'P'
import json, sys
f, tag = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(tag, d["value"], "fps", d["ms_per_step"], "ms", d["stages_ms"], "e2e", d["e2e"]["value"], "tests", d["frame_stats"]["ray_capsule_tests"])
except Exception as e:
    print(tag, "bench failed", e); print(open(f.replace(".json", ".err")).read()[-1500:])
P
}
for w in $WL; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_${TAG}_$w.json 2> gpurun_out/bench_${TAG}_$w.err
  show gpurun_out/bench_${TAG}_$w.json $w
done
for v in $VARIANTS; do
  for w in $WL; do
    LVX_LIB=$PWD/paper_2510_09081_b200/liblvx_b200_$v.so timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_${TAG}_${w}_$v.json 2> gpurun_out/bench_${TAG}_${w}_$v.err
    show gpurun_out/bench_${TAG}_${w}_$v.json $w/$v
  done
done
if [ -z "$NO_NCU" ]; then
for w in $WL; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_render|k_scatter|k_order|k_voxelize|k_shade$|k_visibility' -c 6 --launch-skip ${NCU_SKIP:-0} \
     -o gpurun_out/prof_${TAG}_$w -f python bench.py --workload $w --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_${TAG}_$w.log 2>&1
done
fi
