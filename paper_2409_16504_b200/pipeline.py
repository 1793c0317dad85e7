"""The fused real-time path: point cloud -> P2ENet -> splat planes in one call.

``render_frame`` is ``render_planes(estimate_neural(cloud), cam)`` without
materialising per-point Gaussians: the renderer projects the M0 per-voxel
Gaussians once, sorts points by (voxel depth, index) and composites each
voxel's points as one run (colours per point). Output planes are identical
to the two-step path. This is what ``bench.py`` times.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .gaussians import Camera
from .netplan import NetworkWeights
from .pcio import PointCloud
from .rasterizer import _PLANE_BIT, FrameBuffer, RenderOptions, _alloc_planes
from .sparsenet import ensure_loaded
from .voxelgrid import device_bbox, lattice_scale, stage_cloud


def render_frame(cloud: PointCloud, weights: NetworkWeights, cam: Camera,
                 planes=("rgb", "normal"), background=(0.0, 0.0, 0.0),
                 options: RenderOptions = None, out=None, lane: int = 0) -> FrameBuffer:
    """Cloud -> P2ENet -> planes. ``lane`` selects an independent library
    context (own arena and CUDA graphs): issue frames from different lanes on
    different torch streams and they overlap on the GPU."""
    ctx = ensure_loaded(weights, lane)
    options = options or RenderOptions()
    pos, col = stage_cloud(cloud)
    n = int(pos.shape[0])
    lo_hi = device_bbox(pos, lane)
    s = lattice_scale(n, lo_hi)
    bg = np.ascontiguousarray(np.asarray(background, dtype=np.float64).reshape(3))
    rgb, nrm, dep, trans = out if out is not None else _alloc_planes(cam, planes, pos.device)
    mask = 0
    for p in planes:
        mask |= _PLANE_BIT[p]
    c, o = cam.struct(), options.struct()
    ctx.call("sfb_frame", _lib.ptr(pos), _lib.ptr(col), n, s, lo_hi.ctypes.data_as(_lib.P),
             _lib.ctypes.byref(c), _lib.ctypes.byref(o), mask, bg.ctypes.data_as(_lib.P),
             _lib.ptr(rgb), _lib.ptr(nrm), _lib.ptr(dep), _lib.ptr(trans))
    if rgb is None:
        rgb = torch.zeros((int(cam.height), int(cam.width), 3), dtype=torch.float32,
                          device=pos.device)
    return FrameBuffer(int(cam.width), int(cam.height), rgb, trans, bg, nrm, dep)


def stats(lane: int = 0) -> dict:
    """Sizes of the last call (kept splats, runs, pyramid entries, voxels per level)."""
    return _lib.context(lane=lane).stats()
