"""Diagnostics: GPU P2ENet error statistics vs the float64 oracle on config 1."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from oracle import net as ON, voxel as OV
from paper_2409_16504_b200 import netplan, scenes, sparsenet
from paper_2409_16504_b200.pcio import PointCloud
from paper_2409_16504_b200.voxelgrid import voxelize_adaptive

cloud, _ = scenes.config1()
w = netplan.init_random(netplan.NetworkPlan(), 0)
ov = OV.voxelize(cloud.positions, cloud.colors)
ref_raw = ON.unet(ov, w.as_oracle_layers(), 3, per_voxel=True)
scale = ov["scale_to_world"]
ref = ON.activate(ref_raw, scale)
for mode in ("simt_f32", "tc_tf32x3"):
    sparsenet.set_mode(mode)
    vox = voxelize_adaptive(PointCloud(cloud.positions, cloud.colors))
    raw = sparsenet.unet_forward_voxels(vox, w).cpu().numpy().astype(np.float64)
    d = np.abs(raw - ref_raw)
    print(mode, "raw: max|ref|", np.abs(ref_raw).max(), "max abs err", d.max(),
          "max rel (floor 1e-3*max)", (d / np.maximum(np.abs(ref_raw), 1e-3 * np.abs(ref_raw).max())).max())
    head = sparsenet.activate_head(sparsenet.unet_forward_voxels(vox, w), scale)
    for k, g in (("delta", head.delta), ("sigma", head.sigma), ("quat", head.quat),
                 ("opacity", head.opacity), ("normal", head.normal)):
        g = g.cpu().numpy()
        e = np.abs(g - ref[k])
        i = np.unravel_index(np.argmax(e), e.shape)
        print(f"  {k}: max abs {e.max():.3e} at {i} ref {ref[k][i]:.6g} got {g[i]:.6g}; "
              f"max abs/scale {e.max() / scale:.3e}; rel(max(|ref|,scale)) "
              f"{(e / np.maximum(np.abs(ref[k]), scale)).max():.3e}")
