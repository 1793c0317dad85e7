"""Kernel timeline of frames in flight (torch.profiler / CUPTI, GPU): per kernel
name, total busy time and an SM-occupancy-weighted share (grid size vs 148
SMs x resident CTAs approximated by grid/148 capped at 1) — where the GPU's
capacity goes when lanes overlap."""
import json, sys, collections
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2409_16504_b200 import netplan, scenes
from paper_2409_16504_b200.gaussians import Camera
from paper_2409_16504_b200.pcio import PointCloud
from paper_2409_16504_b200.pipeline import render_frame

lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cloud, views = scenes.config2()
w = netplan.init_random(netplan.NetworkPlan(), 0)
pc = PointCloud(torch.from_numpy(cloud.positions).cuda(), torch.from_numpy(cloud.colors).cuda(), validate=False)
cams = [Camera.of(v) for v in views]
streams = [torch.cuda.Stream() for _ in range(lanes)]
H = W = 1024
outs = [(torch.empty((H, W, 3), dtype=torch.float32, device="cuda"), torch.empty((H, W, 3), dtype=torch.float32, device="cuda"),
         None, torch.empty((H, W), dtype=torch.float32, device="cuda")) for _ in range(lanes)]
def batch(nf):
    for i in range(nf):
        with torch.cuda.stream(streams[i % lanes]):
            render_frame(pc, w, cams[i % 8], out=outs[i % lanes], lane=i % lanes)
    torch.cuda.synchronize()
for _ in range(4):
    batch(2 * lanes)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    batch(4 * lanes)
prof.export_chrome_trace("/tmp/trace.json")
ev = [e for e in json.load(open("/tmp/trace.json"))["traceEvents"] if e.get("cat") == "kernel"]
t0 = min(e["ts"] for e in ev); t1 = max(e["ts"] + e["dur"] for e in ev)
frames = 4 * lanes
agg = collections.defaultdict(lambda: [0.0, 0.0, 0])
for e in ev:
    g = e.get("args", {}).get("grid", [1, 1, 1])
    ctas = g[0] * g[1] * g[2]
    frac = min(1.0, ctas / 148.0)
    name = e["name"].split("(")[0][-50:]
    agg[name][0] += e["dur"]
    agg[name][1] += e["dur"] * frac
    agg[name][2] += 1
tot_w = sum(v[1] for v in agg.values())
print(f"{frames} frames in {t1 - t0:.0f} us = {(t1 - t0) / frames:.1f} us/frame; "
      f"SM-weighted kernel time {tot_w / frames:.1f} us/frame")
for n, (d, wt, c) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{wt / frames:8.1f} us/frame weighted  {d / frames:8.1f} us/frame busy  x{c / frames:4.1f}  {n}")
