mkdir -p gpurun_out
for m in tc_tf32x3 simt_f32 tc_bf16; do
  timeout 300 python bench.py --steps 800 --no-cpu --no-profile --no-e2e --net-mode $m > gpurun_out/mode_$m.json 2>gpurun_out/mode_$m.err
done
