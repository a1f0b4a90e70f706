#!/bin/bash
# Source-level ncu capture of one kernel family.  usage (inside gpurun): bash tools/ncu_one.sh <tag> <workload> <kernel regex> [top lines]
TAG=$1; W=$2; K=$3; TOP=${4:-45}
O=gpurun_out; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$K" --launch-skip ${NCU_SKIP:-12} -c ${NCU_COUNT:-4} \
   -o $O/${TAG}_$W -f python bench.py --workload $W --steps 1 --warmup 3 --no-cpu --no-drop-in --pipeline 1 > $O/${TAG}_$W.log 2>&1
python tools/ncu_summary.py $O/${TAG}_$W.ncu-rep > $O/${TAG}_${W}_summary.txt 2>&1
python tools/ncu_lines.py $O/${TAG}_$W.ncu-rep $TOP > $O/${TAG}_${W}_lines.txt 2>&1
rm -f $O/${TAG}_$W.ncu-rep
cat $O/${TAG}_${W}_summary.txt; head -120 $O/${TAG}_${W}_lines.txt
