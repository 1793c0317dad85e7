#!/bin/bash
# ncu --set full (with source) of one launch each of the named kernels of a
# steady-state config-2 frame (view 0): skip and count are one frame's matches of the
# default regex (14: 9 radix downsweeps + vbuild, vranks, voxel sums, level-0 conv, head).
# usage: bash tools/prof_kernels.sh tag regex
tag=$1; rx=$2
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --lanes 1 --no-e2e --no-cpu --no-profile --view 0"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$rx" \
  --launch-skip 28 -c 14 -f -o gpurun_out/prof_k_$tag $B > gpurun_out/ncu_k_$tag.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_k_$tag.log
