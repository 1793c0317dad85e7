#!/bin/bash
# GPU-box pass: full -m gpu suite, smoke, parity report, short bench.
# usage (repo root, under gpurun): bash tools/gpu_check.sh tag [pytest-args...]
tag=${1:-x}; shift
mkdir -p gpurun_out
nproc > gpurun_out/nproc_$tag.txt; lscpu | grep "Model name" >> gpurun_out/nproc_$tag.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread -p no:cacheprovider "$@" \
  > gpurun_out/gpu_tests_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$tag.log
