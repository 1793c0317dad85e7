"""Gaussian-parameter error statistics of estimate_neural vs the oracle (GPU)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import net as ON
from paper_2409_16504_b200 import netplan, scenes, sparsenet
from paper_2409_16504_b200.estimators import estimate_neural
from paper_2409_16504_b200.pcio import PointCloud

which = sys.argv[1] if len(sys.argv) > 1 else "c5"
cloud, _ = {"c1": scenes.config1, "c2": scenes.config2, "c3": scenes.config3, "c5": scenes.config5}[which]()
w = netplan.init_random(netplan.NetworkPlan(), 0)
est = ON.estimate(cloud.positions, cloud.colors, w.as_oracle_layers(), 3)
for mode in (sys.argv[2].split(",") if len(sys.argv) > 2 else ("tc_tf32x3", "simt_f32")):
    sparsenet.set_mode(mode)
    sp = estimate_neural(PointCloud(cloud.positions, cloud.colors), w)
    scale = est["vox"]["scale_to_world"]
    g = lambda k: getattr(sp, k).detach().cpu().numpy()
    r = np.abs(g("scales") - est["scales"]) / (1e-3 * np.maximum(np.abs(est["scales"]), 1e-3 * scale))
    d = np.abs(g("centers") - est["centers"]) / (1e-3 * scale)
    print(mode, which, "sigma: worst ratio", r.max(), "violations", int((r > 1).sum()), "of", r.size,
          "| delta: worst ratio", d.max(), int((d > 1).sum()))
    i = np.unravel_index(np.argmax(r), r.shape)
    print("  worst sigma", g("scales")[i], est["scales"][i], "scale", scale)
    for k in ("quaternions", "opacities", "normals"):
        e = np.abs(g(k) - est[k])
        print("  ", k, "max abs", e.max(), "violations", int((e > 1e-3).sum()))
    del sp
    torch.cuda.empty_cache()
