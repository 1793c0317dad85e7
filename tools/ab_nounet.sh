mkdir -p gpurun_out
for v in "" _nounet _nocomp; do
  SFB_LIB_PATH=paper_2409_16504_b200/_build/libsfb200$v.so timeout 300 python bench.py --steps 800 --no-cpu --no-profile --no-e2e > gpurun_out/ab$v.json 2>gpurun_out/ab$v.err
done
