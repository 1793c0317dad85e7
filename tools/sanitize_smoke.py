"""A small fused frame + render_pose + backward + kNN for compute-sanitizer runs."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2409_16504_b200 import netplan, scenes, service
from paper_2409_16504_b200.estimators import estimate_neural, nearest_neighbors
from paper_2409_16504_b200.gaussians import Camera
from paper_2409_16504_b200.pcio import PointCloud
from paper_2409_16504_b200.pipeline import render_frame
from paper_2409_16504_b200.rasterizer import render_backward

cloud, views = scenes.config1(n_dirs=3000)
w = netplan.init_random(netplan.NetworkPlan(), 0)
pc = PointCloud(cloud.positions, cloud.colors)
v = views[0]
v.width = v.height = 48
v.cx = v.cy = 24.0
v.fx = v.fy = 24.0 / np.tan(np.radians(30.0))
cam = Camera.of(v)
for _ in range(3):   # eager, capture, replay
    fb = render_frame(pc, w, cam)
sp = estimate_neural(pc, w)
service.render_pose(sp, service.CameraPose(cam, "relit"))
render_backward(sp, cam, np.ones((48, 48, 3)))
nearest_neighbors(cloud.positions[:500], 8)
torch.cuda.synchronize()
print("ok", float(fb.rgb.sum()))
