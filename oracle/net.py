"""Oracle: P2ENet forward (sparse conv, pruned transposed conv, head) in float64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Restates
``splatforge/sparsenet.py:187-341`` and ``estimators.py:214-231``. A network
is a list of layer dicts ``{kind, kernel, cin, cout, w (float32), b (float32)}``
in the reference's forward order (sparsenet.py:108-118).
"""
from __future__ import annotations

import numpy as np

from . import voxel as V

HEAD = 14


def conv(coords, keys, feats, stride, layer, relu=True, nbr=None):
    """out = b + sum_taps feats[nbr] @ W[tap], taps in (dz,dy,dx) order (sparsenet.py:187-214)."""
    k, cin, cout = layer["kernel"], layer["cin"], layer["cout"]
    if nbr is None:
        nbr = V.kernel_map(coords, keys, stride, k)
    w = layer["w"].reshape(k ** 3, cin, cout)
    out = np.empty((coords.shape[0], cout))
    out[:] = layer["b"]
    for t in range(k ** 3):
        hit = nbr[:, t] >= 0
        if hit.any():
            out[hit] += feats[nbr[hit, t]] @ w[t]
    if relu:
        np.maximum(out, 0.0, out=out)
    return out


def tconv(parent_keys, parent_feats, parent_stride, targets, layer, relu=True):
    """Pruned 2x2x2 transposed conv onto the target set (sparsenet.py:217-249)."""
    pidx, tap = V.transposed_map(targets, parent_keys, parent_stride)
    w = layer["w"].reshape(8, layer["cin"], layer["cout"])
    out = np.empty((targets.shape[0], layer["cout"]))
    out[:] = layer["b"]
    for t in range(8):
        sel = (tap == t) & (pidx >= 0)
        if sel.any():
            out[sel] += parent_feats[pidx[sel]] @ w[t]
    if relu:
        np.maximum(out, 0.0, out=out)
    return out


def unet(vox: dict, layers: list, levels: int, per_voxel: bool = False) -> np.ndarray:
    """UNet + head (sparsenet.py:252-287); per-point raw (N,14) unless per_voxel."""
    it = iter(layers)
    coords, keys, feats, stride = vox["coords"], vox["keys"], vox["feats"], 1
    skips = []
    for _ in range(levels):
        feats = conv(coords, keys, feats, stride, next(it))
        skips.append((coords, keys, feats, stride))
        coords, feats, keys = V.pool(coords, feats, stride)
        stride *= 2
    feats = conv(coords, keys, feats, stride, next(it))
    for s_coords, s_keys, s_feats, s_stride in reversed(skips):
        up = tconv(keys, feats, stride, s_coords, next(it))
        coords, keys, stride = s_coords, s_keys, s_stride
        feats = np.concatenate([up, s_feats], axis=1)
    l1, l2 = next(it), next(it)
    hidden = np.maximum(feats @ l1["w"] + l1["b"], 0.0)
    raw = hidden @ l2["w"] + l2["b"]
    return raw if per_voxel else raw[vox["point_to_voxel"]]


def _sigmoid(x):
    """Split-branch logistic (sparsenet.py:301-307)."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def activate(raw: np.ndarray, scale: float) -> dict:
    """Head activations (sparsenet.py:310-341)."""
    raw = np.asarray(raw, dtype=np.float64)
    delta = np.tanh(raw[..., 0:3]) * scale
    sigma = np.maximum(np.logaddexp(0.0, raw[..., 3:6]), 1e-12) * scale
    q = raw[..., 6:10].copy()
    q[..., 0] += 1.0
    qn = np.linalg.norm(q, axis=-1, keepdims=True)
    ident = np.zeros_like(q)
    ident[..., 0] = 1.0
    q = np.where(qn < 1e-12, ident, q / np.maximum(qn, 1e-300))
    opacity = _sigmoid(raw[..., 10])
    n = raw[..., 11:14]
    nn = np.linalg.norm(n, axis=-1, keepdims=True)
    up = np.zeros_like(n)
    up[..., 2] = 1.0
    n = np.where(nn < 1e-8, up, n / np.maximum(nn, 1e-300))
    return dict(delta=delta, sigma=sigma, quat=q, opacity=opacity, normal=n)


def estimate(positions, colors, layers, levels) -> dict:
    """Voxelize -> UNet -> activate -> per-point splats (estimators.py:214-231)."""
    vox = V.voxelize(positions, colors)
    raw = unet(vox, layers, levels)
    head = activate(raw, vox["scale_to_world"])
    centers = V.reconstructed(vox)[vox["point_to_voxel"]] + head["delta"]
    return dict(centers=centers, scales=head["sigma"], quaternions=head["quat"],
                opacities=head["opacity"], colors=np.array(colors, dtype=np.float64),
                normals=head["normal"], vox=vox, raw=raw)
