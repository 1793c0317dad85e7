"""Point cloud -> splats through P2ENet on the GPU (drop-in for the neural path
of the reference estimators.py: EstimatorConfig 22-38, estimate_neural 214-231,
run_estimator 234-245).

Only ``kind="neural"`` is on this repo's hot path; the analytic estimators
(global_isotropic, local_pca) are out of scope and raise.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .gaussians import Splats
from .netplan import NetworkPlan, NetworkWeights, init_random, load_weights
from .pcio import PointCloud
from .sparsenet import ensure_loaded
from .voxelgrid import device_bbox, lattice_scale, stage_cloud

ESTIMATOR_KINDS = ("global_isotropic", "local_pca", "neural")


@dataclass(frozen=True)
class EstimatorConfig:
    kind: str = "neural"
    sigma_multiplier: float = 1.5
    k_neighbors: int = 16
    weights_path: str = None
    default_opacity: float = 1.0

    def __post_init__(self):
        if self.kind not in ESTIMATOR_KINDS:
            raise ValueError(f"unknown estimator kind '{self.kind}'")
        if self.sigma_multiplier <= 0:
            raise ValueError("sigma_multiplier must be positive")
        if self.k_neighbors < 4:
            raise ValueError("k_neighbors must be at least 4")
        if not 0.0 <= self.default_opacity <= 1.0:
            raise ValueError("default_opacity must lie in [0, 1]")


def estimate_neural(cloud: PointCloud, weights: NetworkWeights,
                    cfg: EstimatorConfig = None) -> Splats:
    """Voxelize -> UNet -> activate -> one splat per source point, all on device.

    Centres are the reconstructed voxel positions plus the bounded offset;
    colours are the points' own (estimators.py:214-231)."""
    if weights.plan.encoder_channels[0] != 9:
        raise ValueError(f"input grid has 9 channels, plan expects {weights.plan.encoder_channels[0]}")
    ctx = ensure_loaded(weights)
    pos, col = stage_cloud(cloud)
    n = int(pos.shape[0])
    lo_hi = device_bbox(pos)
    s = lattice_scale(n, lo_hi)
    dev = pos.device
    out = {k: torch.empty((n, w), dtype=torch.float64, device=dev)
           for k, w in (("centers", 3), ("scales", 3), ("quaternions", 4), ("colors", 3),
                        ("normals", 3))}
    opac = torch.empty(n, dtype=torch.float64, device=dev)
    ctx.call("sfb_estimate_neural", _lib.ptr(pos), _lib.ptr(col), n, s,
             lo_hi.ctypes.data_as(_lib.P), _lib.ptr(out["centers"]), _lib.ptr(out["scales"]),
             _lib.ptr(out["quaternions"]), _lib.ptr(opac), _lib.ptr(out["colors"]),
             _lib.ptr(out["normals"]))
    return Splats(out["centers"], out["scales"], out["quaternions"], opac, out["colors"],
                  out["normals"], validate=False)


def run_estimator(cloud: PointCloud, cfg: EstimatorConfig, weights: NetworkWeights = None) -> Splats:
    """Dispatch on cfg.kind (estimators.py:234-245); neural falls back to
    seed-0 random weights when none are given, like the reference."""
    if cfg.kind != "neural":
        raise NotImplementedError(f"estimator '{cfg.kind}' is outside this repo's hot path "
                                  "(only the P2ENet 'neural' estimator is implemented)")
    if weights is None:
        weights = (load_weights(cfg.weights_path) if cfg.weights_path is not None
                   else _default_weights())
    return estimate_neural(cloud, weights, cfg)


_DEFAULT = None


def _default_weights() -> NetworkWeights:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = init_random(NetworkPlan(), 0)
    return _DEFAULT
