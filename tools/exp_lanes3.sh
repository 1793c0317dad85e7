mkdir -p gpurun_out
for L in 8 12 16; do
timeout 300 python bench.py --steps 800 --lanes $L --no-e2e --no-cpu --no-profile > gpurun_out/lanes_$L.json 2> gpurun_out/lanes_$L.err
done
