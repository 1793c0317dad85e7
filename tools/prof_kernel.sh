# ncu --set full of kernels matching a regex in one config-2 frame
# usage: bash tools/prof_kernel.sh '<regex>' <tag> [count] [launch-skip]
re=$1; tag=$2; cnt=${3:-1}; skip=${4:-0}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --lanes 1 --no-e2e --no-cpu --no-profile"
timeout 300 $CMD > gpurun_out/plainfull_$tag.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$re" -s $skip -c $cnt \
  -f -o gpurun_out/prof_$tag $CMD > gpurun_out/ncufull_$tag.log 2>&1
echo "rc=$?" >> gpurun_out/ncufull_$tag.log
