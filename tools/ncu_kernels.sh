#!/bin/bash
# usage (inside gpurun): bash tools/ncu_kernels.sh <tag> <workload> <kernel regex> [count]
# one `ncu --set full` capture of the named kernels of one bench frame (after 3 warm-up frames)
TAG=$1; W=$2; K=$3; C=${4:-4}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$K" --launch-skip ${NCU_SKIP:-0} -c $C \
   -o gpurun_out/prof_${TAG}_$W -f python bench.py --workload $W --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_${TAG}_$W.log 2>&1
tail -3 gpurun_out/ncu_${TAG}_$W.log
