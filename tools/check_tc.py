"""Quick tcgen05-vs-SIMT conv check (GPU)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2409_16504_b200 import netplan, sparsenet, scenes
from paper_2409_16504_b200.voxelgrid import SparseVoxelGrid, voxelize_adaptive
from paper_2409_16504_b200.pcio import PointCloud

rng = np.random.default_rng(0)
for cin, cout, m in [(9, 16, 1000), (16, 32, 700), (32, 64, 300), (64, 128, 449), (3, 5, 200), (64, 16, 5000)]:
    lattice = np.stack(np.meshgrid(*[np.arange(24)] * 3, indexing="ij"), -1).reshape(-1, 3)
    pick = rng.choice(lattice.shape[0], size=m, replace=False)
    grid = SparseVoxelGrid.from_host(lattice[pick], rng.normal(size=(m, cin)).astype(np.float32) * 100)
    spec = netplan.ConvLayerSpec("conv", cin, cout)
    w = rng.uniform(-0.3, 0.3, size=spec.weight_shape).astype(np.float32)
    b = rng.normal(size=cout).astype(np.float32)
    out = {}
    for mode in ("simt_f32", "tc_tf32x3"):
        sparsenet.set_mode(mode)
        out[mode] = sparsenet.sparse_conv(grid, spec, w, b, relu=False).feats.cpu().numpy()
    d = np.abs(out["simt_f32"] - out["tc_tf32x3"])
    print(f"cin {cin} cout {cout} m {m}: max|d| {d.max():.3e} max|ref| {np.abs(out['simt_f32']).max():.3e}", flush=True)
cloud, _ = scenes.config1()
w = netplan.init_random(netplan.NetworkPlan(), 0)
vox = voxelize_adaptive(PointCloud(cloud.positions, cloud.colors))
res = {}
for mode in ("simt_f32", "tc_tf32x3"):
    sparsenet.set_mode(mode)
    res[mode] = sparsenet.unet_forward_voxels(vox, w).cpu().numpy()
print("unet c1 max|d|", np.abs(res["simt_f32"] - res["tc_tf32x3"]).max())
