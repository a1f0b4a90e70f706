#!/bin/bash
# A/B of stage times, serial pass only.  usage: bash tools/ab.sh "<workloads>" "ENV=1" ...   (first run = no env)
WL=$1; shift
for w in $WL; do
  for e in "" "$@"; do
    env $e python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --pipeline 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$w', '[$e]', d['value'], 'fps', d['stages_ms'])"
  done
done
