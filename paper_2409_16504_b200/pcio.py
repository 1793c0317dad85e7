"""Point cloud container (reference pcio.py:39-83) with device residency.

Only the in-memory container is on the hot path: float64 positions (N,3) and
colors (N,3) in [0,1]. Host numpy arrays stay on the host until a pipeline
call stages them (pinned, then one H2D copy); torch CUDA tensors are used in
place.
"""
from __future__ import annotations

import numpy as np
import torch


class EmptyCloudError(ValueError):
    """A cloud with zero points where at least one is required."""


class DegenerateCloudError(ValueError):
    """Geometry without the extent an operation needs (e.g. all points coincident)."""


class PointCloud:
    """positions (N,3) float64 world units; colors (N,3) float64 in [0,1]."""

    def __init__(self, positions, colors, normals=None, validate: bool = True):
        self.positions = _f64(positions)
        self.colors = _f64(colors)
        self.normals = None if normals is None else _f64(normals)
        if self.positions.ndim != 2 or self.positions.shape[1] != 3:
            raise ValueError(f"positions must be (N, 3), got {tuple(self.positions.shape)}")
        if tuple(self.colors.shape) != tuple(self.positions.shape):
            raise ValueError("colors must match positions shape")
        if validate and self.colors.shape[0]:
            lo, hi = float(self.colors.min()), float(self.colors.max())
            if lo < 0.0 or hi > 1.0:
                raise ValueError("color channels must lie in [0, 1]")

    def __len__(self) -> int:
        return int(self.positions.shape[0])

    @property
    def on_device(self) -> bool:
        return isinstance(self.positions, torch.Tensor) and self.positions.is_cuda


def _f64(a):
    if isinstance(a, torch.Tensor):
        return a.to(torch.float64).contiguous()
    return np.ascontiguousarray(a, dtype=np.float64)
