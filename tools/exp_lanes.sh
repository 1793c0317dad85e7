for r in 1 2; do for l in 6 8 10 12; do timeout 300 python bench.py --steps 800 --lanes $l --no-cpu --no-profile --no-e2e > gpurun_out/lanes_$l.$r.json 2>/dev/null; done; done
