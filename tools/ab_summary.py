"""Summarise an A/B run of tools/gpu_perf.sh: per variant, per repetition,
throughput ms/frame, latency ms, eager UNet ms and compositor kernel ms.
usage: python tools/ab_summary.py <tag>"""
import collections
import glob
import json
import sys

tag = sys.argv[1]
res = collections.defaultdict(list)
for f in sorted(glob.glob(f"gpurun_out/ab_{tag}*.json")):
    v = f.split(f"ab_{tag}")[1].rsplit(".", 2)[0] or "(main)"
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        st = d["stages_ms_eager"]
        res[v].append((round(d["ms_per_step"], 4), round(d["latency_ms_per_frame"], 4),
                       round(st["unet"], 4), round(st.get("composite_kernel", 0), 4)))
    except Exception as e:  # noqa: BLE001
        res[v].append(f"error: {str(e)[:60]}")
print("variant      [(throughput ms, latency ms, unet ms, composite ms) per repetition]")
for v, r in res.items():
    print(f"{v:12s}", r)
