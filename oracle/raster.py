"""Oracle: tiled front-to-back splatting (float64), plus the brute-force blend.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). The numpy glue restates
``splatforge/rasterizer.py:99-166`` (_prepare, _compose, render) and
``render_reference`` (rasterizer.py:169-206); the three hot loops run in
``raster_oracle.c`` (restating _raster_kernels.py:20-201), loaded via ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle_raster.so"
Z_NEAR = 0.01          # gaussians.py:21
DILATION = 0.3         # gaussians.py:22
ALPHA_MAX = 0.99       # gaussians.py:23
CUTOFF = 1.0 / 255.0   # _raster_kernels.py:16-17

_lib = None


def build() -> Path:
    """Compile raster_oracle.c (make -C oracle); returns the .so path."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = ctypes.CDLL(str(LIB))
        P, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double
        _lib.oracle_project.argtypes = [P, P, P, I, P, P, D, D, D, D, I, I, D, D] + [P] * 8
        _lib.oracle_bin_count.argtypes = [P, P, P, I, I, I, I, I, I, I, I, P]
        _lib.oracle_bin_count.restype = I
        _lib.oracle_bin_fill.argtypes = [P, P, P, I, I, I, I, I, I, I, I, P, P]
        _lib.oracle_forward.argtypes = [I, I, I, I, I, I, I, P, P, P, P, P, P, P, P, P, P,
                                        D, ctypes.c_int, P, P]
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt=np.float64):
    return np.ascontiguousarray(a, dtype=dt)


def project(centers, quats, scales, cam) -> dict:
    """project_kernel (_raster_kernels.py:20-105) for every splat."""
    centers, quats, scales = _c(centers), _c(quats), _c(scales)
    n = centers.shape[0]
    out = {k: np.zeros(n) for k in ("sx", "sy", "depth", "a", "b", "c", "radius")}
    keep = np.zeros(n, dtype=np.uint8)
    rot, tr = _c(cam.rotation), _c(cam.translation)
    lib().oracle_project(_p(centers), _p(quats), _p(scales), n, _p(rot), _p(tr),
                         float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy),
                         int(cam.width), int(cam.height), Z_NEAR, DILATION,
                         *[_p(out[k]) for k in ("sx", "sy", "depth", "a", "b", "c", "radius")],
                         _p(keep))
    out["keep"] = keep.astype(bool)
    return out


def prepare(splats: dict, cam, mode: str, tile: int = 16, ty_window=None, tx_window=None) -> dict:
    """Depth sort, inverse covariance, alpha-support radius, CSR tile lists
    (rasterizer.py:99-130)."""
    pr = project(splats["centers"], splats["quaternions"], splats["scales"], cam)
    kept = np.nonzero(pr["keep"])[0]
    source = kept[np.argsort(pr["depth"][kept], kind="stable")]
    sx, sy, depth = pr["sx"][source], pr["sy"][source], pr["depth"][source]
    cov = np.stack([pr["a"][source], pr["b"][source], pr["c"][source]], axis=1)
    det = cov[:, 0] * cov[:, 2] - cov[:, 1] ** 2
    inv = np.stack([cov[:, 2] / det, -cov[:, 1] / det, cov[:, 0] / det], axis=1)
    opac = _c(np.asarray(splats["opacities"], dtype=np.float64)[source])
    mid = 0.5 * (cov[:, 0] + cov[:, 2])
    gap = np.sqrt(np.maximum(0.25 * (cov[:, 0] - cov[:, 2]) ** 2 + cov[:, 1] ** 2, 0.0))
    lam = np.maximum(mid + gap, 0.0)
    support = 2.0 * np.log(np.maximum(255.0 * opac, 1e-300))
    radius = np.sqrt(np.maximum(support, 0.0) * lam) + 1e-9
    ntx = -(-int(cam.width) // tile)
    nty = -(-int(cam.height) // tile)
    lo, hi = (0, nty) if ty_window is None else ty_window
    xlo, xhi = (0, ntx) if tx_window is None else tx_window
    offsets = np.zeros(ntx * nty + 1, dtype=np.int64)
    sx, sy, radius = _c(sx), _c(sy), _c(radius)
    e = lib().oracle_bin_count(_p(sx), _p(sy), _p(radius), sx.size, tile, ntx, nty, lo, hi,
                               xlo, xhi, _p(offsets))
    ids = np.empty(e, dtype=np.int64)
    lib().oracle_bin_fill(_p(sx), _p(sy), _p(radius), sx.size, tile, ntx, nty, lo, hi,
                          xlo, xhi, _p(offsets), _p(ids))
    if mode == "rgb":
        attr = np.asarray(splats["colors"], dtype=np.float64)[source]
    elif mode == "normal":
        attr = np.asarray(splats["normals"], dtype=np.float64)[source]
    else:
        attr = np.zeros((source.size, 3))
        attr[:, 0] = depth
    return dict(source=source, sx=sx, sy=sy, depth=depth, cov=cov, inv=_c(inv), opac=opac,
                radius=radius, attr=_c(attr), offsets=offsets, ids=ids, ntx=ntx, nty=nty,
                window=(lo, hi))


def compose(out, trans, mode, background):
    """Planes from the blend accumulators (rasterizer.py:140-149, 53-55)."""
    bg = np.asarray(background, dtype=np.float64).reshape(3)
    t = np.clip(trans, 0.0, 1.0)
    if mode == "rgb":
        return dict(rgb=out + trans[:, :, None] * bg, transmittance=t)
    if mode == "normal":
        norms = np.linalg.norm(out, axis=2, keepdims=True)
        normal = np.divide(out, norms, out=np.zeros_like(out), where=norms > 0.0)
        return dict(rgb=np.zeros_like(out), normal=normal, transmittance=t)
    return dict(rgb=np.zeros_like(out), depth=out[:, :, 0].copy(), transmittance=t)


def render(splats: dict, cam, mode="rgb", background=(0.0, 0.0, 0.0), tile=16,
           alpha_max=ALPHA_MAX, terminate=True, ty_window=None, prep=None, tx_window=None) -> dict:
    """Tiled render (rasterizer.py:152-166); returns planes plus the prepared CSR.
    ty_window / tx_window restrict the binned tiles to a crop (tests and the
    bounded CPU sample): pixels outside it are left unrendered."""
    if prep is None:
        prep = prepare(splats, cam, mode, tile, ty_window, tx_window)
    w, h = int(cam.width), int(cam.height)
    out = np.zeros((h, w, 3))
    trans = np.ones((h, w))
    lo, hi = prep["window"]
    inv = prep["inv"]
    lib().oracle_forward(w, h, tile, prep["ntx"], prep["nty"], lo, hi, _p(prep["offsets"]),
                         _p(prep["ids"]), _p(prep["sx"]), _p(prep["sy"]), _p(prep["radius"]),
                         _p(_c(inv[:, 0])), _p(_c(inv[:, 1])), _p(_c(inv[:, 2])),
                         _p(prep["opac"]), _p(prep["attr"]), float(alpha_max), int(bool(terminate)),
                         _p(out), _p(trans))
    fb = compose(out, trans, mode, background)
    fb["prep"] = prep
    return fb


def render_bruteforce(splats: dict, cam, mode="rgb", background=(0.0, 0.0, 0.0),
                      alpha_max=ALPHA_MAX) -> dict:
    """Per-pixel blend over every projected splat, no tiles, no termination
    (render_reference, rasterizer.py:169-206; projection as gaussians.py:221-263)."""
    pr = project(splats["centers"], splats["quaternions"], splats["scales"], cam)
    idx = np.nonzero(pr["keep"])[0]
    order = idx[np.lexsort((idx, pr["depth"][idx]))]
    w, h = int(cam.width), int(cam.height)
    xs, ys = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    out = np.zeros((h, w, 3))
    trans = np.ones((h, w))
    for i in order:
        a, b, c = pr["a"][i], pr["b"][i], pr["c"][i]
        det = a * c - b * b
        dx = xs - pr["sx"][i]
        dy = ys - pr["sy"][i]
        q = (c * dx * dx - 2.0 * b * dx * dy + a * dy * dy) / det
        alpha = np.minimum(splats["opacities"][i] * np.exp(-0.5 * q), alpha_max)
        live = alpha >= CUTOFF
        if mode == "rgb":
            attr = splats["colors"][i]
        elif mode == "normal":
            attr = splats["normals"][i]
        else:
            attr = np.array([pr["depth"][i], 0.0, 0.0])
        out += np.where(live, trans * alpha, 0.0)[:, :, None] * attr
        trans = np.where(live, trans * (1.0 - alpha), trans)
    return compose(out, trans, mode, background)


def to_rgba(plane, transmittance) -> np.ndarray:
    """RGBA8 quantisation with coverage alpha (service.py:116-120)."""
    rgb = np.clip(np.rint(plane * 255.0), 0, 255).astype(np.uint8)
    a = np.clip(np.rint((1.0 - transmittance) * 255.0), 0, 255).astype(np.uint8)
    return np.concatenate([rgb, a[:, :, None]], axis=2)


def relight(normal, rgb, transmittance, light, ambient, diffuse) -> np.ndarray:
    """Lambertian late shading with background pass-through (rasterizer.py:209-226)."""
    lam = np.maximum(normal @ np.asarray(light, dtype=np.float64), 0.0)
    shaded = rgb * (ambient + diffuse * lam)[:, :, None]
    return np.clip(np.where((transmittance > 0.999)[:, :, None], rgb, shaded), 0.0, 1.0)
