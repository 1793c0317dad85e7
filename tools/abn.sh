# A/B over library variants: bash tools/abn.sh "" _x _y ...  (interleaved, 2 rounds)
mkdir -p gpurun_out
for r in 1 2; do
for v in "$@"; do
  SFB_LIB_PATH=paper_2409_16504_b200/_build/libsfb200$v.so timeout 300 python bench.py --steps 800 --no-cpu --no-profile --no-e2e > gpurun_out/abn$v.$r.json 2>gpurun_out/abn$v.$r.err
done; done
