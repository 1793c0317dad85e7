"""Host-side cost of one render_frame call (GPU): bbox read-back, Python glue, sfb_frame enqueue."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2409_16504_b200 import _lib, netplan, scenes
from paper_2409_16504_b200.gaussians import Camera
from paper_2409_16504_b200.pcio import PointCloud
from paper_2409_16504_b200.pipeline import render_frame
from paper_2409_16504_b200.voxelgrid import device_bbox, lattice_scale

cloud, views = scenes.config2()
w = netplan.init_random(netplan.NetworkPlan(), 0)
pc = PointCloud(torch.from_numpy(cloud.positions).cuda(), torch.from_numpy(cloud.colors).cuda(), validate=False)
cam = Camera.of(views[0])
for _ in range(5):
    render_frame(pc, w, cam)
torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
for _ in range(N):
    lo_hi = device_bbox(pc.positions)
t1 = time.perf_counter()
print(f"device_bbox (incl. sync) {1e3*(t1-t0)/N:.3f} ms/call")
t0 = time.perf_counter()
for _ in range(N):
    lattice_scale(len(cloud), lo_hi)
t1 = time.perf_counter()
print(f"lattice_scale {1e3*(t1-t0)/N:.4f} ms/call")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(N):
    render_frame(pc, w, cam)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"render_frame enqueue {1e3*(t1-t0)/N:.3f} ms/call, total {1e3*(t2-t0)/N:.3f} ms/frame (1 lane)")
