#!/bin/bash
# round-2 GPU check: new tests, tiled emulation on C4, culling-active C2, alpha sweep of C3, reference arm
O=gpurun_out; mkdir -p $O; T=r02b
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > $O/${T}_tests_gpu.log; cat $O/${T}_tests_gpu.log
for G in 2 4 8; do
  timeout 600 python bench.py --workload c4 --emulate-world $G --steps 5 --warmup 3 --no-cpu > $O/${T}_emu_c4_g$G.json 2> $O/${T}_emu_c4_g$G.err
  python - $O/${T}_emu_c4_g$G.json <<'P'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print("emu", d["emulated"]["world"], d["value"], "fps")
    for r in d["emulated"]["ranks"]: print("  ", r["rank"], r["own_stage_ms_sum"], r["stages_ms"], r["stats"]["fragments"])
except Exception as e: print("FAILED", e); print(open(sys.argv[1].replace(".json",".err")).read()[-2000:])
P
done
for a in 0.1 0.5; do
  timeout 600 python bench.py --workload c3 --alpha $a --steps 10 --warmup 3 --no-cpu > $O/${T}_bench_c3_a$a.json 2> $O/${T}_bench_c3_a$a.err
  tail -c 900 $O/${T}_bench_c3_a$a.json | head -c 400; echo
done
timeout 600 python bench.py --workload c2thick --steps 10 --warmup 3 --no-cpu > $O/${T}_bench_c2thick.json 2> $O/${T}_bench_c2thick.err
python - $O/${T}_bench_c2thick.json <<'P'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print("c2thick", d["value"], d["stages_ms"], d["frame_stats"])
P
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/${T}_bench_c2_reference.json 2> $O/${T}_bench_c2_reference.err
cut -c1-1200 $O/${T}_bench_c2_reference.json
