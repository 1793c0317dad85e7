mkdir -p gpurun_out
timeout 300 python tools/diag_composite.py > gpurun_out/diag_comp.txt 2>&1
for L in 1 2 4 8; do
timeout 300 python bench.py --steps 400 --lanes $L --no-e2e --no-cpu --no-profile > gpurun_out/lanes_$L.json 2> gpurun_out/lanes_$L.err
done
timeout 300 python tools/host_overhead.py > gpurun_out/host_overhead.txt 2>&1
