"""Per-view compositor counters on config 2 (GPU diagnostics)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2409_16504_b200 import _lib, netplan, scenes
from paper_2409_16504_b200.gaussians import Camera
from paper_2409_16504_b200.pcio import PointCloud
from paper_2409_16504_b200.pipeline import render_frame, stats

cloud, views = scenes.config2()
w = netplan.init_random(netplan.NetworkPlan(), 0)
pc = PointCloud(torch.from_numpy(cloud.positions).cuda(), torch.from_numpy(cloud.colors).cuda())
ctx = _lib.context()
ctx.lib.sfb_set_graphs(ctx.handle, 0)
cnt = torch.zeros(4096 * 4, dtype=torch.int64, device="cuda")
for k, v in enumerate(views):
    cam = Camera.of(v)
    render_frame(pc, w, cam)
    torch.cuda.synchronize()
    cnt.zero_()
    ctx.lib.sfb_set_debug_counters(ctx.handle, _lib.ptr(cnt))
    fb = render_frame(pc, w, cam)
    torch.cuda.synchronize()
    ctx.lib.sfb_set_debug_counters(ctx.handle, _lib.P(0))
    c = cnt.view(4096, 4).cpu().numpy()
    T = fb.transmittance.cpu().numpy()
    st = stats()
    print(f"view {k}: windows/tile mean {c[:,0].mean():.2f} max {c[:,0].max()}, entries/tile mean "
          f"{c[:,1].mean():.1f} max {c[:,1].max()}, alpha evals/px {c[:,2].mean()/256:.1f} max {c[:,2].max()/256:.1f}, "
          f"point blends/px {c[:,3].mean()/256:.1f}, "
          f"unsat px {(T >= 1/255).mean():.3f}, runs {st['runs']} fine {st['fine_entries']} super {st['super_entries']} "
          f"global {st['global_entries']}", flush=True)
