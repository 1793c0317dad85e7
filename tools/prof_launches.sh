# launch list of one config-2 frame: plain run, then ncu (gpu__time_duration per launch)
tag=${1:-x}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --lanes 1 --no-e2e --no-cpu --no-profile"
timeout 300 $CMD > gpurun_out/plain_$tag.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control ${CACHE:-all} -c 400 --csv \
  --log-file gpurun_out/launches_$tag.csv $CMD > gpurun_out/ncu_$tag.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_$tag.log
