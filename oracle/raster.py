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
        _lib.oracle_forward_stream.argtypes = [I, I, I, I] + [P] * 9 + [D, ctypes.c_int, P, P, P]
        _lib.oracle_backward.argtypes = [I, I, I, I, I, P, P, P, P, P, P, P, P, P, D,
                                         ctypes.c_int, ctypes.c_int, P, P, P, P, P, P]
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


def render_banded(splats: dict, cam, mode="rgb", background=(0.0, 0.0, 0.0), tile=16,
                  alpha_max=ALPHA_MAX, terminate=True, band_rows=8) -> dict:
    """The reference render (rasterizer.py:152-166) over the WHOLE frame with
    bounded memory: _prepare's projection, sort and support radius once, then
    bin_tiles + forward_kernel per band of ``band_rows`` tile rows (the full
    random-init config-2 CSR would hold ~1.6e9 int64 ids). Every tile is
    binned and blended exactly as in one full pass; planes are identical to
    ``render``. This is the CPU reference arm's timed frame (bench.py)."""
    prep = prepare(splats, cam, mode, tile, ty_window=(0, 0))
    w, h = int(cam.width), int(cam.height)
    ntx, nty = prep["ntx"], prep["nty"]
    out = np.zeros((h, w, 3))
    trans = np.ones((h, w))
    sx, sy, radius = prep["sx"], prep["sy"], prep["radius"]
    inv = prep["inv"]
    ia, ib, ic = _c(inv[:, 0]), _c(inv[:, 1]), _c(inv[:, 2])
    offsets = np.zeros(ntx * nty + 1, dtype=np.int64)
    for lo in range(0, nty, band_rows):
        hi = min(nty, lo + band_rows)
        e = lib().oracle_bin_count(_p(sx), _p(sy), _p(radius), sx.size, tile, ntx, nty, lo, hi,
                                   0, ntx, _p(offsets))
        ids = np.empty(e, dtype=np.int64)
        lib().oracle_bin_fill(_p(sx), _p(sy), _p(radius), sx.size, tile, ntx, nty, lo, hi, 0, ntx,
                              _p(offsets), _p(ids))
        lib().oracle_forward(w, h, tile, ntx, nty, lo, hi, _p(offsets), _p(ids), _p(sx), _p(sy),
                             _p(radius), _p(ia), _p(ib), _p(ic), _p(prep["opac"]),
                             _p(prep["attr"]), float(alpha_max), int(bool(terminate)), _p(out),
                             _p(trans))
        del ids
    return compose(out, trans, mode, background)


def render_stream(splats: dict, cam, modes=("rgb", "normal"), background=(0.0, 0.0, 0.0),
                  tile=16, alpha_max=ALPHA_MAX, terminate=True) -> dict:
    """Full-frame tiled render (rasterizer.py:152-166) of one or two attribute
    modes in one pass, without materialising the CSR: the per-tile entry
    lists are generated in rank order on the fly (oracle_forward_stream), so
    the random-init frames of configs 2-5 render in seconds. Planes are
    identical to ``render`` (pinned against it and the reference goldens in
    tests/test_oracle.py)."""
    prep = prepare(splats, cam, modes[0], tile, ty_window=(0, 0))   # sort + radius, no bins
    src = prep["source"]
    attrs = []
    for m in modes:
        if m == "rgb":
            attrs.append(_c(np.asarray(splats["colors"], dtype=np.float64)[src]))
        elif m == "normal":
            attrs.append(_c(np.asarray(splats["normals"], dtype=np.float64)[src]))
        else:
            a = np.zeros((src.size, 3))
            a[:, 0] = prep["depth"]
            attrs.append(a)
    w, h = int(cam.width), int(cam.height)
    outs = [np.zeros((h, w, 3)) for _ in modes]
    trans = np.ones((h, w))
    inv = prep["inv"]
    lib().oracle_forward_stream(w, h, tile, src.size, _p(prep["sx"]), _p(prep["sy"]),
                                _p(prep["radius"]), _p(_c(inv[:, 0])), _p(_c(inv[:, 1])),
                                _p(_c(inv[:, 2])), _p(prep["opac"]), _p(attrs[0]),
                                _p(attrs[1]) if len(modes) > 1 else None, float(alpha_max),
                                int(bool(terminate)), _p(outs[0]),
                                _p(outs[1]) if len(modes) > 1 else None, _p(trans))
    fb = {}
    for m, out in zip(modes, outs):
        fb.update({k: v for k, v in compose(out, trans, m, background).items()
                   if k in (m, "transmittance")})
    fb["source"] = src
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


def _quat_to_rotmat(q):
    """gaussians.py:160-177, batched."""
    q = np.asarray(q, dtype=np.float64)
    norm = np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = np.moveaxis(q / norm, -1, 0)
    r = np.empty(q.shape[:-1] + (3, 3), dtype=np.float64)
    r[..., 0, 0] = 1 - 2 * (y * y + z * z)
    r[..., 0, 1] = 2 * (x * y - w * z)
    r[..., 0, 2] = 2 * (x * z + w * y)
    r[..., 1, 0] = 2 * (x * y + w * z)
    r[..., 1, 1] = 1 - 2 * (x * x + z * z)
    r[..., 1, 2] = 2 * (y * z - w * x)
    r[..., 2, 0] = 2 * (x * z - w * y)
    r[..., 2, 1] = 2 * (y * z + w * x)
    r[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return r


def render_backward(splats: dict, cam, upstream, mode="rgb", background=(0.0, 0.0, 0.0),
                    tile=16, alpha_max=ALPHA_MAX, terminate=True) -> dict:
    """Analytic gradients of render() (rasterizer.py:229-354): per-entry slots from
    backward_kernel, the ordered entry->splat reduction (np.add.at), then the chain
    rule through the inverse covariance, EWA Jacobian, rotation and normalisation."""
    modes = ("rgb", "normal", "depth")
    background = np.asarray(background, dtype=np.float64).reshape(3)
    h, w = int(cam.height), int(cam.width)
    if mode == "depth":
        upstream = np.asarray(upstream, dtype=np.float64)
        if upstream.shape == (h, w):
            lifted = np.zeros((h, w, 3))
            lifted[:, :, 0] = upstream
            upstream = lifted
    upstream = np.ascontiguousarray(upstream, dtype=np.float64)
    prep = prepare(splats, cam, mode, tile)
    k = len(prep["source"])
    entries = prep["ids"].shape[0]
    g_mu = np.zeros((entries, 2))
    g_q = np.zeros((entries, 3))
    g_opac = np.zeros(entries)
    g_attr = np.zeros((entries, 3))
    inv = prep["inv"]
    lib().oracle_backward(w, h, tile, prep["ntx"], prep["nty"], _p(prep["offsets"]),
                          _p(prep["ids"]), _p(prep["sx"]), _p(prep["sy"]), _p(_c(inv[:, 0])),
                          _p(_c(inv[:, 1])), _p(_c(inv[:, 2])), _p(prep["opac"]), _p(prep["attr"]),
                          float(alpha_max), int(bool(terminate)), modes.index(mode),
                          _p(background), _p(upstream), _p(g_mu), _p(g_q), _p(g_opac), _p(g_attr))
    d_mu = np.zeros((k, 2))
    d_qf = np.zeros((k, 3))
    d_op = np.zeros(k)
    d_at = np.zeros((k, 3))
    np.add.at(d_mu, prep["ids"], g_mu)
    np.add.at(d_qf, prep["ids"], g_q)
    np.add.at(d_op, prep["ids"], g_opac)
    np.add.at(d_at, prep["ids"], g_attr)
    n = np.asarray(splats["opacities"]).shape[0]
    out = dict(d_centers=np.zeros((n, 3)), d_scales=np.zeros((n, 3)),
               d_quaternions=np.zeros((n, 4)), d_opacities=np.zeros(n),
               d_colors=np.zeros((n, 3)), d_normals=np.zeros((n, 3)))
    if k == 0:
        return out
    src = prep["source"]
    inv_m = np.empty((k, 2, 2))
    inv_m[:, 0, 0] = inv[:, 0]
    inv_m[:, 0, 1] = inv_m[:, 1, 0] = inv[:, 1]
    inv_m[:, 1, 1] = inv[:, 2]
    g_inv = np.empty((k, 2, 2))
    g_inv[:, 0, 0] = d_qf[:, 0]
    g_inv[:, 0, 1] = g_inv[:, 1, 0] = 0.5 * d_qf[:, 1]
    g_inv[:, 1, 1] = d_qf[:, 2]
    g_cov = -np.einsum("kij,kjl,klm->kim", inv_m, g_inv, inv_m)
    rot_c = np.asarray(cam.rotation, dtype=np.float64)
    centers = np.asarray(splats["centers"], dtype=np.float64)
    p_cam = centers[src] @ rot_c.T + np.asarray(cam.translation, dtype=np.float64)
    x, y, z = p_cam[:, 0], p_cam[:, 1], p_cam[:, 2]
    fx, fy = float(cam.fx), float(cam.fy)
    jac = np.zeros((k, 2, 3))
    jac[:, 0, 0] = fx / z
    jac[:, 0, 2] = -fx * x / (z * z)
    jac[:, 1, 1] = fy / z
    jac[:, 1, 2] = -fy * y / (z * z)
    a2 = jac @ rot_c
    g_s3 = np.einsum("kji,kjl,klm->kim", a2, g_cov, a2)
    quats = np.asarray(splats["quaternions"], dtype=np.float64)[src]
    scales = np.asarray(splats["scales"], dtype=np.float64)[src]
    rot = _quat_to_rotmat(quats)
    sigma3 = np.einsum("kji,kj,kjl->kil", rot, scales * scales, rot)
    m_cam = np.einsum("ij,kjl,ml->kim", rot_c, sigma3, rot_c)
    g_jac = 2.0 * np.einsum("kij,kjl,klm->kim", g_cov, jac, m_cam)
    d_pcam = np.zeros((k, 3))
    d_pcam[:, 0] = g_jac[:, 0, 2] * (-fx / (z * z))
    d_pcam[:, 1] = g_jac[:, 1, 2] * (-fy / (z * z))
    d_pcam[:, 2] = (g_jac[:, 0, 0] * (-fx / (z * z)) + g_jac[:, 0, 2] * (2.0 * fx * x / z ** 3)
                    + g_jac[:, 1, 1] * (-fy / (z * z)) + g_jac[:, 1, 2] * (2.0 * fy * y / z ** 3))
    d_pcam[:, 0] += d_mu[:, 0] * fx / z
    d_pcam[:, 1] += d_mu[:, 1] * fy / z
    d_pcam[:, 2] += d_mu[:, 0] * (-fx * x / (z * z)) + d_mu[:, 1] * (-fy * y / (z * z))
    if mode == "depth":
        d_pcam[:, 2] += d_at[:, 0]
    out["d_centers"][src] = d_pcam @ rot_c
    g_d = np.einsum("kij,kjl,kml->kim", rot, g_s3, rot)
    out["d_scales"][src] = 2.0 * scales * np.stack([g_d[:, 0, 0], g_d[:, 1, 1], g_d[:, 2, 2]], axis=1)
    g_r = 2.0 * (scales * scales)[:, :, None] * (rot @ g_s3)
    qn = np.linalg.norm(quats, axis=1, keepdims=True)
    w_, qx, qy, qz = (quats / qn).T
    zero = np.zeros(k)
    drdq = np.empty((k, 4, 3, 3))
    drdq[:, 0] = 2.0 * np.stack([zero, -qz, qy, qz, zero, -qx, -qy, qx, zero], axis=1).reshape(k, 3, 3)
    drdq[:, 1] = 2.0 * np.stack([zero, qy, qz, qy, -2 * qx, -w_, qz, w_, -2 * qx], axis=1).reshape(k, 3, 3)
    drdq[:, 2] = 2.0 * np.stack([-2 * qy, qx, w_, qx, zero, qz, -w_, qz, -2 * qy], axis=1).reshape(k, 3, 3)
    drdq[:, 3] = 2.0 * np.stack([-2 * qz, -w_, qx, w_, -2 * qz, qy, qx, qy, zero], axis=1).reshape(k, 3, 3)
    d_qhat = np.einsum("kij,kqij->kq", g_r, drdq)
    qhat = quats / qn
    out["d_quaternions"][src] = (d_qhat - qhat * np.sum(qhat * d_qhat, axis=1, keepdims=True)) / qn
    out["d_opacities"][src] = d_op
    if mode == "rgb":
        out["d_colors"][src] = d_at
    elif mode == "normal":
        out["d_normals"][src] = d_at
    return out
