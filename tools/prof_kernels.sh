#!/bin/bash
# ncu --set full (with source) of the launches matching a regex over one
# steady-state config-2 frame (view 0): skip = 2 frames' matches, count = one
# frame's (the caller passes the per-frame match count).
# usage: bash tools/prof_kernels.sh tag regex per_frame_matches
tag=$1; rx=$2; k=${3:-14}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --lanes 1 --no-e2e --no-cpu --no-profile --view 0"
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$rx" \
  --launch-skip $((2 * k)) -c $k -f -o gpurun_out/prof_k_$tag $B > gpurun_out/ncu_k_$tag.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_k_$tag.log
