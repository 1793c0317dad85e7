"""Golden outputs of the reference's analytic estimators (estimators.py:41-211,
_neighbors.py:33-128): exact kNN with index tie-breaks, local-PCA and global
isotropic splats. Build container only:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb \\
        python tests/golden/make_golden_estimators.py

Seeded clouds generated here (a noisy sphere shell with duplicated points for
exact ties, and an integer lattice patch); every output comes from the
reference and is stored in tests/golden/estimators.npz.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from splatforge._neighbors import nearest_neighbors  # noqa: E402
from splatforge.estimators import EstimatorConfig, estimate_global, estimate_local_pca  # noqa: E402
from splatforge.pcio import PointCloud  # noqa: E402

OUT = Path(__file__).resolve().parent / "estimators.npz"
KEYS = ("centers", "scales", "quaternions", "opacities", "colors", "normals")


def clouds():
    rng = np.random.default_rng(31)
    u = rng.normal(size=(1400, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    shell = u * (20.0 + rng.normal(scale=0.3, size=(1400, 1))) + [5.0, -3.0, 8.0]
    shell = np.concatenate([shell, shell[:60]])          # exact duplicates -> distance ties
    g = np.stack(np.meshgrid(np.arange(12), np.arange(12), np.arange(3), indexing="ij"), -1)
    lattice = g.reshape(-1, 3).astype(np.float64) * [1.0, 1.0, 2.5]   # many equal distances
    return {"shell": shell, "lattice": lattice}


def main():
    out = {}
    rng = np.random.default_rng(5)
    for name, pos in clouds().items():
        col = rng.random(pos.shape)
        out[f"{name}_positions"] = pos
        out[f"{name}_colors"] = col
        d2, idx = nearest_neighbors(pos, 16)
        out[f"{name}_knn_d2"], out[f"{name}_knn_idx"] = d2, idx
        cloud = PointCloud(pos, col)
        for kind, fn in (("pca", estimate_local_pca), ("global", estimate_global)):
            sp = fn(cloud, EstimatorConfig(kind="local_pca" if kind == "pca" else "global_isotropic"))
            for k in KEYS:
                out[f"{name}_{kind}_{k}"] = getattr(sp, k)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
