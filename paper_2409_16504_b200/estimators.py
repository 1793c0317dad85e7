"""Point cloud -> splats on the GPU (drop-in for the reference estimators.py:
EstimatorConfig 22-38, estimate_global 147-163, estimate_local_pca 166-211,
estimate_neural 214-231, run_estimator 234-245) and the exact kNN of
_neighbors.py (nearest_neighbors 85-122, mean_nn_distance 125-128).

The neural path (P2ENet) is the hot path; the analytic estimators share the
render back end: exact kNN on a device uniform grid,
per-point covariance + closed-form 3x3 eigen frames (csrc/knn.cu).
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
    kind: str = "local_pca"
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


def nearest_neighbors(positions, k: int):
    """(N, k) squared distances and int64 indices of each point's k nearest
    others, ascending with the index as tie-break (_neighbors.py:85-122);
    bit-identical to the reference."""
    pos = positions if isinstance(positions, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(positions, dtype=np.float64))
    pos = pos.to("cuda", torch.float64).contiguous()
    if pos.ndim != 2 or pos.shape[1] != 3:
        raise ValueError(f"positions must be (N, 3), got {tuple(pos.shape)}")
    n = int(pos.shape[0])
    if k < 1:
        raise ValueError("k must be at least 1")
    if k >= n:
        raise ValueError(f"{k} neighbors need at least {k + 1} points, got {n}")
    d2 = torch.empty((n, k), dtype=torch.float64, device=pos.device)
    idx = torch.empty((n, k), dtype=torch.int64, device=pos.device)
    _lib.context().call("sfb_knn", _lib.ptr(pos), n, k, _lib.ptr(d2), _lib.ptr(idx))
    return d2, idx


def _mean_first_distance(d2: torch.Tensor) -> float:
    """mean of sqrt(d2[:, 0]) with numpy's summation (the reference's d-bar)."""
    n, k = d2.shape
    dist = torch.empty(n, dtype=torch.float64, device=d2.device)
    _lib.context().call("sfb_nn_distance", _lib.ptr(d2), n, k, _lib.ptr(dist))
    return float(dist.cpu().numpy().mean())


def mean_nn_distance(positions) -> float:
    """Mean distance to the single nearest neighbour, d-bar (_neighbors.py:125-128)."""
    d2, _ = nearest_neighbors(positions, 1)
    return _mean_first_distance(d2)


def _cloud_normals(cloud: PointCloud, pos: torch.Tensor) -> torch.Tensor:
    if cloud.normals is not None:
        n = cloud.normals
        return (n if isinstance(n, torch.Tensor) else torch.from_numpy(n)).to(pos.device, torch.float64).clone()
    out = torch.zeros_like(pos)
    out[:, 2] = 1.0
    return out


def _colors(cloud: PointCloud, pos: torch.Tensor) -> torch.Tensor:
    c = cloud.colors
    return (c if isinstance(c, torch.Tensor) else torch.from_numpy(c)).to(pos.device, torch.float64).clone()


def estimate_global(cloud: PointCloud, cfg: EstimatorConfig) -> Splats:
    """One isotropic splat per point, sized by the mean nearest-neighbour
    distance (estimators.py:147-163)."""
    from .pcio import DegenerateCloudError
    pos, _ = stage_cloud(cloud)
    n = int(pos.shape[0])
    if n < 2:
        raise ValueError("global estimation needs at least 2 points")
    d_bar = mean_nn_distance(pos)
    if d_bar == 0.0:
        raise DegenerateCloudError("all points coincident; density scale is zero")
    sigma = cfg.sigma_multiplier * d_bar
    quats = torch.zeros((n, 4), dtype=torch.float64, device=pos.device)
    quats[:, 0] = 1.0
    return Splats(pos.clone(), torch.full((n, 3), sigma, dtype=torch.float64, device=pos.device),
                  quats, torch.full((n,), float(cfg.default_opacity), dtype=torch.float64,
                                    device=pos.device),
                  _colors(cloud, pos), _cloud_normals(cloud, pos), validate=False)


def estimate_local_pca(cloud: PointCloud, cfg: EstimatorConfig) -> Splats:
    """Anisotropic splats from the covariance of each point's k nearest
    neighbours (estimators.py:166-211): eigen frame rows in ascending
    eigenvalue order with the reference's sign rules, scales
    sigma_multiplier*sqrt(lambda) clamped below at 0.1*d-bar, normal = the
    smallest-eigenvalue direction flipped away from the centroid."""
    from .pcio import DegenerateCloudError
    pos, _ = stage_cloud(cloud)
    n = int(pos.shape[0])
    k = cfg.k_neighbors
    if n < k + 1:
        raise ValueError(f"local PCA needs at least {k + 1} points, got {n}")
    d2, idx = nearest_neighbors(pos, k)
    d_bar = _mean_first_distance(d2)
    if d_bar == 0.0:
        raise DegenerateCloudError("all points coincident; density scale is zero")
    host = cloud.positions
    centroid = (host.detach().cpu().numpy() if isinstance(host, torch.Tensor) else host).mean(axis=0)
    centroid = np.ascontiguousarray(centroid, dtype=np.float64)
    scales = torch.empty((n, 3), dtype=torch.float64, device=pos.device)
    quats = torch.empty((n, 4), dtype=torch.float64, device=pos.device)
    normals = torch.empty((n, 3), dtype=torch.float64, device=pos.device)
    _lib.context().call("sfb_local_pca", _lib.ptr(pos), n, k, _lib.ptr(idx),
                        float(cfg.sigma_multiplier), d_bar, centroid.ctypes.data_as(_lib.P),
                        _lib.ptr(scales), _lib.ptr(quats), _lib.ptr(normals))
    return Splats(pos.clone(), scales, quats,
                  torch.full((n,), float(cfg.default_opacity), dtype=torch.float64, device=pos.device),
                  _colors(cloud, pos), normals, validate=False)


def run_estimator(cloud: PointCloud, cfg: EstimatorConfig, weights: NetworkWeights = None) -> Splats:
    """Dispatch on cfg.kind (estimators.py:234-245); neural falls back to
    seed-0 random weights when none are given, like the reference."""
    if cfg.kind == "global_isotropic":
        return estimate_global(cloud, cfg)
    if cfg.kind == "local_pca":
        return estimate_local_pca(cloud, cfg)
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
