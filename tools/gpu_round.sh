#!/bin/bash
# One GPU-box pass: GPU tests, default bench, ncu launch list, ncu --set full of k_composite.
# usage (from the repo root, under gpurun): bash tools/gpu_round.sh [tag]
tag=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q --timeout 240 --timeout-method thread > gpurun_out/gpu_tests_$tag.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$tag.log
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
echo "bench rc=$?" >> gpurun_out/bench_$tag.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv \
  --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 1 --lanes 1 \
  --no-e2e --no-cpu --no-profile > gpurun_out/ncu_$tag.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_$tag.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite \
  --launch-skip 12 -c 1 -f -o gpurun_out/prof_comp_$tag python bench.py --steps 2 --warmup 1 \
  --lanes 1 --no-e2e --no-cpu --no-profile > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full_$tag.log
timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers \
  --clock-control none --cache-control none -c 400 --csv --log-file gpurun_out/smlaunch_$tag.csv \
  python bench.py --steps 2 --warmup 1 --lanes 1 --no-e2e --no-cpu --no-profile > gpurun_out/ncu_sm_$tag.log 2>&1
echo "ncu sm rc=$?" >> gpurun_out/ncu_sm_$tag.log
