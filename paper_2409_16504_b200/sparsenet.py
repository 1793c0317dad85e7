"""P2ENet on the GPU: sparse convolutions, pruned transposed convolutions,
UNet forward and head activations (drop-in for the reference sparsenet.py).

The network description, ``init_random`` and the P2EN weight format live in
``netplan.py`` (re-exported here under the reference names); the arithmetic
runs in libsfb200 (csrc/net.cu, csrc/conv_tc.cu). Features inside the network
are float32 (fp32 accumulation); the head activations and everything that
feeds the renderer are float64.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .netplan import (HEAD_CHANNELS, ConvLayerSpec, NetworkPlan, NetworkWeights,  # noqa: F401
                      WeightFormatError, WeightShapeError, WeightTruncationError, init_random,
                      load_weights, save_weights, weights_from_bytes, weights_to_bytes)
from .voxelgrid import SparseVoxelGrid, VoxelizedCloud

MODES = {"simt_f32": _lib.NET_SIMT_F32, "tc_tf32x3": _lib.NET_TC_TF32X3,
         "tc_bf16": _lib.NET_TC_BF16, "simt_f64": _lib.NET_SIMT_F64}
_mode = "tc_tf32x3"


def set_mode(mode: str) -> None:
    """Select the network arithmetic for every lane: 'tc_tf32x3' (tcgen05, tf32
    hi/lo split, fp32-accurate: the default), 'tc_bf16' (tcgen05, single bf16
    operands, fp32 accumulation: fast, outside the 1e-3 parameter bound),
    'simt_f32' (FFMA) or 'simt_f64' (float64 features, the reference's own
    arithmetic on the FP64 pipe: the end-to-end exactness mode)."""
    global _mode
    if mode not in MODES:
        raise ValueError(f"unknown network mode {mode!r}; expected one of {tuple(MODES)}")
    _mode = mode
    for ctx in _lib.all_contexts():
        _apply_mode(ctx)


def _apply_mode(ctx) -> None:
    if getattr(ctx, "net_mode", None) != _mode:
        if ctx.lib.sfb_net_set_mode(ctx.handle, MODES[_mode]) != _lib.SFB_OK:
            raise ValueError(f"cannot select network mode {_mode!r}")
        ctx.net_mode = _mode


def ensure_loaded(weights: NetworkWeights, lane: int = 0) -> _lib.Context:
    """Upload a network once per context (re-upload when a different object is passed)."""
    ctx = _lib.context(lane=lane)
    _apply_mode(ctx)
    if ctx.net_token is not weights:
        blob = weights_to_bytes(weights)
        buf = np.frombuffer(blob, dtype=np.uint8)
        ctx.call("sfb_net_load", buf.ctypes.data_as(_lib.P), len(blob))
        ctx.net_token = weights
    return ctx


def _check_layer(grid, spec, kind, weights, bias):
    if spec.kind != kind:
        raise ValueError(f"expected a {kind} spec, got '{spec.kind}'")
    if grid.channel_count != spec.in_channels:
        raise ValueError(f"grid has {grid.channel_count} channels, layer expects {spec.in_channels}")
    w = np.ascontiguousarray(weights, dtype=np.float32)
    b = np.ascontiguousarray(bias, dtype=np.float32)
    if w.shape != spec.weight_shape:
        raise ValueError(f"weights must be {spec.weight_shape}, got {w.shape}")
    if b.shape != (spec.out_channels,):
        raise ValueError(f"bias must be ({spec.out_channels},), got {b.shape}")
    ctx = _lib.context()
    _apply_mode(ctx)
    ctx.call("sfb_layer_set", 0 if kind == "conv" else 1, spec.kernel, spec.in_channels,
             spec.out_channels, w.ctypes.data_as(_lib.P), b.ctypes.data_as(_lib.P))
    return ctx


def sparse_conv(grid: SparseVoxelGrid, spec: ConvLayerSpec, weights, bias,
                relu: bool = False) -> SparseVoxelGrid:
    """Stride-1 conv at the occupied sites (sparsenet.py:187-214)."""
    ctx = _check_layer(grid, spec, "conv", weights, bias)
    m = len(grid)
    f = grid.feats.to(torch.float32).contiguous()
    out = torch.empty((m, spec.out_channels), dtype=torch.float32, device=grid.coords.device)
    ctx.call("sfb_sparse_conv", -1, _lib.ptr(grid.coords), _lib.ptr(f), m, grid.stride,
             int(relu), _lib.ptr(out))
    return SparseVoxelGrid(grid.coords, out, grid.stride, grid.scale_to_world, grid.keys)


def transposed_conv_pruned(grid: SparseVoxelGrid, spec: ConvLayerSpec, weights, bias,
                           target_occupancy, relu: bool = False) -> SparseVoxelGrid:
    """2x2x2 upsampling onto an explicit target set (sparsenet.py:217-249)."""
    ctx = _check_layer(grid, spec, "transposed_conv", weights, bias)
    if grid.stride < 2:
        raise ValueError("transposed conv needs a stride >= 2 grid to subdivide")
    child = grid.stride // 2
    if isinstance(target_occupancy, torch.Tensor):
        t = target_occupancy.to(device=grid.coords.device, dtype=torch.int32).contiguous()
    else:
        tn = np.ascontiguousarray(np.atleast_2d(target_occupancy), dtype=np.int64)
        if tn.ndim != 2 or tn.shape[1] != 3:
            raise ValueError(f"target occupancy must be (K, 3), got {tn.shape}")
        if tn.size and (tn % child != 0).any():
            raise ValueError(f"target coordinates must be multiples of {child}")
        t = torch.from_numpy(tn.astype(np.int32)).to(grid.coords.device)
    mt = int(t.shape[0])
    f = grid.feats.to(torch.float32).contiguous()
    out = torch.empty((mt, spec.out_channels), dtype=torch.float32, device=grid.coords.device)
    ctx.call("sfb_transposed_conv", -1, _lib.ptr(grid.coords), _lib.ptr(f), len(grid),
             grid.stride, _lib.ptr(t), mt, int(relu), _lib.ptr(out))
    return SparseVoxelGrid(t, out, child, grid.scale_to_world)


def unet_forward_voxels(vox: VoxelizedCloud, weights: NetworkWeights) -> torch.Tensor:
    """UNet + head, one raw 14-vector per VOXEL (M0,14): float32, float64 in
    'simt_f64' mode."""
    plan = weights.plan
    if vox.grid.channel_count != plan.encoder_channels[0]:
        raise ValueError(f"input grid has {vox.grid.channel_count} channels, "
                         f"plan expects {plan.encoder_channels[0]}")
    ctx = ensure_loaded(weights)
    m = len(vox.grid)
    dt = torch.float64 if _mode == "simt_f64" else torch.float32
    raw = torch.empty((m, HEAD_CHANNELS), dtype=dt, device=vox.grid.coords.device)
    feats = vox.grid.feats.to(torch.float64).contiguous()
    ctx.call("sfb_unet_forward", _lib.ptr(vox.grid.coords), _lib.ptr(feats), m, _lib.ptr(raw))
    return raw


def unet_forward(vox: VoxelizedCloud, weights: NetworkWeights) -> torch.Tensor:
    """Per-point raw head outputs (N,14) (sparsenet.py:252-287, broadcast at :287)."""
    return unet_forward_voxels(vox, weights)[vox.point_to_voxel.long()]


@dataclass(eq=False)
class HeadOutput:
    delta: torch.Tensor
    sigma: torch.Tensor
    quat: torch.Tensor
    opacity: torch.Tensor
    normal: torch.Tensor


def activate_head(raw, voxel_scale: float) -> HeadOutput:
    """Bounded splat parameters from raw head outputs (sparsenet.py:310-341):
    float64 in (the reference's dtype; float32 raw from the UNet widens
    exactly), float64 out."""
    if isinstance(raw, torch.Tensor):
        r = raw.to(device="cuda", dtype=torch.float64)
    else:
        r = torch.from_numpy(np.asarray(raw, dtype=np.float64)).cuda()
    if r.shape[-1] != HEAD_CHANNELS:
        raise ValueError(f"raw head output must have {HEAD_CHANNELS} channels")
    if voxel_scale <= 0:
        raise ValueError("voxel_scale must be positive")
    lead = tuple(r.shape[:-1])
    r = r.reshape(-1, HEAD_CHANNELS).contiguous()
    m = int(r.shape[0])
    dev = r.device
    d = torch.empty((m, 3), dtype=torch.float64, device=dev)
    s = torch.empty((m, 3), dtype=torch.float64, device=dev)
    q = torch.empty((m, 4), dtype=torch.float64, device=dev)
    o = torch.empty(m, dtype=torch.float64, device=dev)
    n = torch.empty((m, 3), dtype=torch.float64, device=dev)
    _lib.context().call("sfb_activate_head", _lib.ptr(r), m, float(voxel_scale), _lib.ptr(d),
                        _lib.ptr(s), _lib.ptr(q), _lib.ptr(o), _lib.ptr(n))
    return HeadOutput(d.reshape(lead + (3,)), s.reshape(lead + (3,)), q.reshape(lead + (4,)),
                      o.reshape(lead), n.reshape(lead + (3,)))
