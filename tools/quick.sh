# quick GPU check: gpu tests + short bench (+ optional extra command)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 240 --timeout-method thread > gpurun_out/quick_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick_tests.log
timeout 300 python bench.py --steps 400 --no-cpu --no-profile > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
timeout 300 python tools/diag_composite.py > gpurun_out/quick_diag.txt 2>&1
