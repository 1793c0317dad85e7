#!/bin/bash
# Perf pass on the GPU box: A/B bench over library variants (interleaved),
# compositor counters, ncu launch list + SM cost, ncu --set full of k_composite.
# usage: [AB_ONLY=1] bash tools/gpu_perf.sh tag "" _base ...   (variants = _build/libsfb200<v>.so)
tag=$1; shift
mkdir -p gpurun_out
for r in 1 2; do
for v in "$@"; do
  SFB_LIB_PATH=paper_2409_16504_b200/_build/libsfb200$v.so timeout 300 python bench.py --steps 800 --no-cpu --no-profile --no-e2e > gpurun_out/ab_${tag}$v.$r.json 2>gpurun_out/ab_${tag}$v.$r.err
done; done
[ -n "$AB_ONLY" ] && exit 0
timeout 300 python tools/diag_composite.py > gpurun_out/diag_comp_$tag.txt 2>&1
B="python bench.py --steps 2 --warmup 1 --lanes 1 --no-e2e --no-cpu --no-profile"
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers \
  --clock-control none --cache-control none -c 400 --csv --log-file gpurun_out/smlaunch_$tag.csv $B > gpurun_out/ncu_sm_$tag.log 2>&1
echo "ncu sm rc=$?" >> gpurun_out/ncu_sm_$tag.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite \
  --launch-skip 12 -c 1 -f -o gpurun_out/prof_comp_$tag $B > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full_$tag.log
