# A/B: the committed build (_base) against the working tree's build, interleaved
mkdir -p gpurun_out
for r in 1 2; do
for v in _base ""; do
  SFB_LIB_PATH=paper_2409_16504_b200/_build/libsfb200$v.so timeout 300 python bench.py --steps 800 --no-cpu --no-profile --no-e2e > gpurun_out/ab2$v.$r.json 2>gpurun_out/ab2$v.$r.err
done; done
