"""Tile-based front-to-back splatting on the GPU (drop-in for the reference
rasterizer.py: RenderOptions 25-29, FrameBuffer 32-55, render 152-166).

``render`` keeps the reference signature and per-mode semantics;
``render_planes`` renders several planes (rgb + normal [+ depth]) in ONE pass
(alpha and transmittance do not depend on the blended attribute, so every
plane is identical to its single-mode render). Planes are float32 CUDA
tensors; ``FrameBuffer.numpy()`` brings them to the host.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .gaussians import ALPHA_MAX, Camera, Splats

_MODES = ("rgb", "normal", "depth")
_PLANE_BIT = {"rgb": _lib.PLANE_RGB, "normal": _lib.PLANE_NORMAL, "depth": _lib.PLANE_DEPTH}


@dataclass
class RenderOptions:
    tile_size: int = 16
    alpha_max: float = ALPHA_MAX
    early_termination: bool = True

    def struct(self) -> _lib.RenderOptions_t:
        if not 1 <= int(self.tile_size) <= 32:
            raise ValueError("tile_size must be in [1, 32]")
        return _lib.RenderOptions_t(int(self.tile_size), int(bool(self.early_termination)),
                                    float(self.alpha_max))


@dataclass(eq=False)
class FrameBuffer:
    """Output planes of one render (device float32); transmittance = T_final."""

    width: int
    height: int
    rgb: torch.Tensor
    transmittance: torch.Tensor
    background: np.ndarray
    normal: torch.Tensor = None
    depth: torch.Tensor = None

    def numpy(self) -> dict:
        out = {"rgb": self.rgb, "transmittance": self.transmittance, "normal": self.normal,
               "depth": self.depth}
        return {k: (None if v is None else v.detach().cpu().numpy().astype(np.float64))
                for k, v in out.items()}


def _check(cam: Camera, mode):
    if mode not in _MODES:
        raise ValueError(f"mode must be one of {_MODES}, got {mode!r}")
    if cam.width < 1 or cam.height < 1:
        raise ValueError("image must have positive dimensions")


def _alloc_planes(cam: Camera, planes, device):
    h, w = int(cam.height), int(cam.width)
    rgb = torch.empty((h, w, 3), dtype=torch.float32, device=device) if "rgb" in planes else None
    nrm = torch.empty((h, w, 3), dtype=torch.float32, device=device) if "normal" in planes else None
    dep = torch.empty((h, w), dtype=torch.float32, device=device) if "depth" in planes else None
    trans = torch.empty((h, w), dtype=torch.float32, device=device)
    return rgb, nrm, dep, trans


def render_planes(splats: Splats, cam: Camera, planes=("rgb", "normal"),
                  background=(0.0, 0.0, 0.0), options: RenderOptions = None,
                  out=None) -> FrameBuffer:
    """One compositing pass producing every requested plane (+ transmittance)."""
    for p in planes:
        _check(cam, p)
    options = options or RenderOptions()
    bg = np.ascontiguousarray(np.asarray(background, dtype=np.float64).reshape(3))
    dev = splats.centers.device
    rgb, nrm, dep, trans = out if out is not None else _alloc_planes(cam, planes, dev)
    mask = 0
    for p in planes:
        mask |= _PLANE_BIT[p]
    s, c, o = splats.struct(), cam.struct(), options.struct()
    _lib.context().call("sfb_render", _lib.ctypes.byref(s), _lib.ctypes.byref(c),
                        _lib.ctypes.byref(o), mask, bg.ctypes.data_as(_lib.P), _lib.ptr(rgb),
                        _lib.ptr(nrm), _lib.ptr(dep), _lib.ptr(trans))
    if rgb is None:
        rgb = torch.zeros((int(cam.height), int(cam.width), 3), dtype=torch.float32, device=dev)
    return FrameBuffer(int(cam.width), int(cam.height), rgb, trans, bg, nrm, dep)


def render(splats: Splats, cam: Camera, mode: str = "rgb", background=(0.0, 0.0, 0.0),
           options: RenderOptions = None) -> FrameBuffer:
    """Tiled front-to-back splatting of one mode (rasterizer.py:152-166)."""
    _check(cam, mode)
    return render_planes(splats, cam, (mode,), background, options)


def project(splats: Splats, cam: Camera) -> dict:
    """project_kernel outputs per splat (_raster_kernels.py:20-105), float64."""
    n = len(splats)
    dev = splats.centers.device
    out = {k: torch.empty(n, dtype=torch.float64, device=dev)
           for k in ("sx", "sy", "depth", "a", "b", "c", "radius")}
    keep = torch.empty(n, dtype=torch.uint8, device=dev)
    s, c = splats.struct(), cam.struct()
    _lib.context().call("sfb_project", _lib.ctypes.byref(s), _lib.ctypes.byref(c), 0.01, 0.3,
                        *[_lib.ptr(out[k]) for k in ("sx", "sy", "depth", "a", "b", "c", "radius")],
                        _lib.ptr(keep))
    out["keep"] = keep.bool()
    return out


def prepare_debug(splats: Splats, cam: Camera, tile_size: int = 16) -> dict:
    """The reference CSR of _prepare/bin_tiles (rasterizer.py:99-130): rank->splat
    ``source``, alpha-support ``radius`` per rank, tile ``offsets`` and ``ids``.
    For parity checks only — the render path never materialises this."""
    n = len(splats)
    dev = splats.centers.device
    ntx = -(-int(cam.width) // tile_size)
    nty = -(-int(cam.height) // tile_size)
    source = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    radius = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    offsets = torch.empty(ntx * nty + 1, dtype=torch.int64, device=dev)
    k, e = _lib.I64(0), _lib.I64(0)
    s, c = splats.struct(), cam.struct()
    ctx = _lib.context()
    ctx.call("sfb_prepare_debug", _lib.ctypes.byref(s), _lib.ctypes.byref(c), tile_size,
             _lib.ptr(source), _lib.ptr(radius), _lib.ptr(offsets), _lib.P(0), 0,
             _lib.ctypes.byref(k), _lib.ctypes.byref(e))
    ids = torch.empty(max(e.value, 1), dtype=torch.int64, device=dev)
    ctx.call("sfb_prepare_debug", _lib.ctypes.byref(s), _lib.ctypes.byref(c), tile_size,
             _lib.ptr(source), _lib.ptr(radius), _lib.ptr(offsets), _lib.ptr(ids), e.value,
             _lib.ctypes.byref(k), _lib.ctypes.byref(e))
    return dict(source=source[:k.value], radius=radius[:k.value], offsets=offsets,
                ids=ids[:e.value], ntx=ntx, nty=nty)


def relight(normal_fb: FrameBuffer, rgb_fb: FrameBuffer, light_dir, ambient: float,
            diffuse: float) -> torch.Tensor:
    """Lambertian late shading (rasterizer.py:209-226) on device planes."""
    if normal_fb.normal is None:
        raise ValueError("normal_fb must carry a normal plane")
    light = np.asarray(light_dir, dtype=np.float64).reshape(3)
    if abs(np.linalg.norm(light) - 1.0) > 1e-6:
        raise ValueError("light_dir must be unit length")
    n = normal_fb.normal.to(torch.float64)
    lam = torch.clamp(n @ torch.from_numpy(light).to(n.device), min=0.0)
    rgb = rgb_fb.rgb.to(torch.float64)
    shaded = rgb * (ambient + diffuse * lam)[:, :, None]
    passthrough = (rgb_fb.transmittance > 0.999)[:, :, None]
    return torch.clamp(torch.where(passthrough, rgb, shaded), 0.0, 1.0)


@dataclass(eq=False)
class RenderGradients:
    """Loss partials per input splat (rasterizer.py:59-68); culled splats hold zeros."""

    d_centers: torch.Tensor
    d_scales: torch.Tensor
    d_quaternions: torch.Tensor
    d_opacities: torch.Tensor
    d_colors: torch.Tensor
    d_normals: torch.Tensor


def render_backward(splats: Splats, cam: Camera, upstream, mode: str = "rgb",
                    background=(0.0, 0.0, 0.0), options: RenderOptions = None) -> RenderGradients:
    """Analytic gradients of render() w.r.t. every splat parameter
    (rasterizer.py:229-354). ``upstream`` is dL/d(plane): (H, W, 3) for rgb and
    normal, (H, W) for depth (numpy or CUDA tensor)."""
    _check(cam, mode)
    options = options or RenderOptions()
    if int(options.tile_size) > 16:
        raise ValueError("render_backward supports tile_size <= 16")
    dev = splats.centers.device
    h, w = int(cam.height), int(cam.width)
    up = upstream if isinstance(upstream, torch.Tensor) else torch.from_numpy(np.asarray(upstream))
    up = up.to(device=dev, dtype=torch.float64)
    if mode == "depth" and tuple(up.shape) == (h, w):
        lifted = torch.zeros((h, w, 3), dtype=torch.float64, device=dev)
        lifted[:, :, 0] = up
        up = lifted
    if tuple(up.shape) != (h, w, 3):
        raise ValueError("upstream shape must match the rendered plane")
    up = up.contiguous()
    n = len(splats)
    z = lambda *shape: torch.zeros(shape, dtype=torch.float64, device=dev)
    g = RenderGradients(z(n, 3), z(n, 3), z(n, 4), z(n), z(n, 3), z(n, 3))
    bg = np.ascontiguousarray(np.asarray(background, dtype=np.float64).reshape(3))
    s, c, o = splats.struct(), cam.struct(), options.struct()
    _lib.context().call("sfb_render_backward", _lib.ctypes.byref(s), _lib.ctypes.byref(c),
                        _lib.ctypes.byref(o), _MODES.index(mode), bg.ctypes.data_as(_lib.P),
                        _lib.ptr(up), _lib.ptr(g.d_centers), _lib.ptr(g.d_scales),
                        _lib.ptr(g.d_quaternions), _lib.ptr(g.d_opacities), _lib.ptr(g.d_colors),
                        _lib.ptr(g.d_normals))
    return g
