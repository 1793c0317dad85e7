# per-launch duration and SM-active cycles of one config-2 frame (what each kernel costs in
# SM time, the resource concurrent frame lanes compete for)
tag=${1:-x}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --lanes 1 --no-e2e --no-cpu --no-profile"
timeout 300 $CMD > gpurun_out/plain_$tag.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers \
  --clock-control none --cache-control none -c 400 --csv \
  --log-file gpurun_out/smlaunch_$tag.csv $CMD > gpurun_out/ncu_sm_$tag.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_sm_$tag.log
