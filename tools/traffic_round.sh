#!/bin/bash
# Re-capture the per-kernel `ncu --set full` summaries and profiles/ncu_traffic.json (with the hash of csrc/) after a
# kernel change.   usage (inside gpurun): bash tools/traffic_round.sh <tag> [workloads]
TAG=${1:-rXX}; shift; WL=${@:-c2 c3 c4 c2thick}
O=gpurun_out; mkdir -p $O; cp profiles/ncu_traffic.json $O/ncu_traffic.json 2>/dev/null
for w in $WL; do
  timeout 1200 ncu --set full --clock-control none \
     -k regex:'k_render|k_scatter|k_order$|k_voxelize|k_shade$|k_visibility|k_march|k_upload|k_pack_mip1|k_mip_next|k_solid|k_dilate|k_scan|k_resolve|k_nzmask|k_march_levels|k_need_list|k_ormip$|k_brick_flags|k_super_flags|k_superbrick_shadow' \
     --launch-skip ${NCU_SKIP:-66} -c 32 -o $O/${TAG}_all_$w -f python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --no-drop-in --pipeline 1 > $O/${TAG}_ncu_$w.log 2>&1
  python tools/ncu_summary.py $O/${TAG}_all_$w.ncu-rep $O/ncu_traffic.json $w > $O/${TAG}_ncu_full_${w}_summary.txt 2>&1
  rm -f $O/${TAG}_all_$w.ncu-rep
  head -3 $O/${TAG}_ncu_full_${w}_summary.txt
done
