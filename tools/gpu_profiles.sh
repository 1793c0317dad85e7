#!/bin/bash
# ncu evidence of one config-2 frame (one GPU; each command exits 0 without ncu first):
# launch list with SM cost, --set full of k_composite, tcgen05 conv metrics.
# usage (repo root, under gpurun): bash tools/gpu_profiles.sh tag
tag=${1:-x}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --lanes 1 --no-e2e --no-cpu --no-profile --view 0"
timeout 300 $B > gpurun_out/prof_plain_$tag.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers \
  --clock-control none --cache-control none -c 400 --csv --log-file gpurun_out/smlaunch_$tag.csv $B > gpurun_out/ncu_sm_$tag.log 2>&1
echo "ncu sm rc=$?" >> gpurun_out/ncu_sm_$tag.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite \
  --launch-skip 12 -c 1 -f -o gpurun_out/prof_comp_$tag $B > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full_$tag.log
bash tools/conv_profile.sh $tag
