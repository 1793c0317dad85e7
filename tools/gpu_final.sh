#!/bin/bash
# Round checkpoint on one GPU box: full -m gpu suite, smoke, the default bench
# (and its reference arm), every config's bench line, then the ncu evidence
# (launch list + SM cost, --set full of k_composite, conv tensor metrics).
# usage (repo root, under gpurun): bash tools/gpu_final.sh tag
tag=${1:-x}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread -p no:cacheprovider \
  > gpurun_out/gpu_tests_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$tag.log
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
echo "bench rc=$?" >> gpurun_out/bench_$tag.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
for c in c1 c3 c4 c5; do
  timeout 600 python bench.py --config $c > gpurun_out/bc_${tag}_$c.json 2> gpurun_out/bc_${tag}_$c.err
done
bash tools/gpu_profiles.sh $tag
