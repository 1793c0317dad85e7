#!/bin/bash
# ncu of every tcgen05 conv launch of one config-2 frame (tensor pipe, TMEM,
# duration, DRAM bytes, occupancy) + a SASS census of the shipped library.
# usage (repo root, under gpurun): bash tools/conv_profile.sh tag
tag=${1:-x}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --lanes 1 --no-e2e --no-cpu --no-profile --view 0"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_active,sm__inst_executed_pipe_tmem.sum,smsp__inst_executed_pipe_tmem.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__occupancy_limit_shared_mem,launch__cluster_dim_x \
  -k regex:"k_conv" --clock-control none --cache-control none -c 60 --csv --log-file gpurun_out/conv_ncu_$tag.csv $B > gpurun_out/conv_ncu_$tag.log 2>&1
echo "ncu conv rc=$?" >> gpurun_out/conv_ncu_$tag.log
