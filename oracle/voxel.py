"""Oracle: voxel keys, density-1 voxelization, pooling, neighbour (kernel) maps.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Restates
``splatforge/voxelgrid.py`` and the lookup half of ``sparsenet.py``.
"""
from __future__ import annotations

import numpy as np

BIAS = 1 << 20          # voxelgrid.py:18-19
AXIS_BITS = 21


def pack(coords: np.ndarray) -> np.ndarray:
    """(z, y, x)-monotone int64 key, 21 bits per axis (voxelgrid.py:22-27)."""
    c = np.asarray(coords, dtype=np.int64)
    if c.size and (np.abs(c) >= BIAS).any():
        raise ValueError(f"voxel coordinates must satisfy |c| < {BIAS}")
    return ((c[:, 2] + BIAS) << (2 * AXIS_BITS)) | ((c[:, 1] + BIAS) << AXIS_BITS) | (c[:, 0] + BIAS)


def unpack(keys: np.ndarray) -> np.ndarray:
    """Inverse of pack (voxelgrid.py:30-37)."""
    k = np.asarray(keys, dtype=np.int64)
    m = (1 << AXIS_BITS) - 1
    return np.stack([(k & m) - BIAS, ((k >> AXIS_BITS) & m) - BIAS,
                     ((k >> (2 * AXIS_BITS)) & m) - BIAS], axis=1).astype(np.int32)


def canonical(coords: np.ndarray, feats: np.ndarray):
    """Rows re-sorted by key, duplicates rejected (voxelgrid.py:72-79)."""
    keys = pack(coords)
    perm = np.argsort(keys, kind="stable")
    keys = keys[perm]
    if keys.size > 1 and np.any(keys[1:] == keys[:-1]):
        raise ValueError("duplicate voxel coordinates")
    return (np.ascontiguousarray(np.asarray(coords, dtype=np.int32)[perm]),
            np.ascontiguousarray(np.asarray(feats, dtype=np.float64)[perm]), keys)


def lookup(sorted_keys: np.ndarray, query: np.ndarray) -> np.ndarray:
    """Row of each query coordinate or -1; out-of-range queries miss.

    searchsorted lookup (voxelgrid.py:88-94) behind the range clip of
    ``_lookup_clipped`` (sparsenet.py:178-184).
    """
    q = np.asarray(query, dtype=np.int64)
    rows = np.full(q.shape[0], -1, dtype=np.int64)
    ok = np.all(np.abs(q) < BIAS, axis=1)
    if not ok.any() or sorted_keys.size == 0:
        return rows
    qk = pack(q[ok])
    pos = np.minimum(np.searchsorted(sorted_keys, qk), sorted_keys.size - 1)
    rows[ok] = np.where(sorted_keys[pos] == qk, pos, -1)
    return rows


def voxel_scale(positions: np.ndarray) -> float:
    """s = (N / V_bbox)^(1/3) with the reference's float ops (voxelgrid.py:133-141)."""
    n = positions.shape[0]
    if n < 2:
        raise ValueError("voxelization needs at least 2 points")
    extent = positions.max(axis=0) - positions.min(axis=0)
    volume = float(np.prod(extent))
    if volume <= 0.0:
        raise ValueError("bbox volume is zero; cannot pick a density-1 scale")
    return (n / volume) ** (1.0 / 3.0)


def voxelize(positions: np.ndarray, colors: np.ndarray) -> dict:
    """Density-1 voxelization (voxelgrid.py:125-168).

    Returns coords (M,3) int32 in key order, feats (M,9) float64
    [centroid/s, mean colour, clipped residual], keys, scale_to_world = 1/s,
    point_to_voxel (N,), source_order (N,) and source_offsets (M+1,).
    """
    positions = np.ascontiguousarray(positions, dtype=np.float64)
    colors = np.ascontiguousarray(colors, dtype=np.float64)
    s = voxel_scale(positions)
    scaled = positions * s
    keys = pack(np.floor(scaled).astype(np.int64))
    ukeys, inv, cnt = np.unique(keys, return_inverse=True, return_counts=True)
    m = ukeys.size
    # ordered per-voxel sums: np.add.at walks points in increasing index
    csum = np.zeros((m, 3))
    np.add.at(csum, inv, scaled)
    centroid = csum / cnt[:, None]
    rsum = np.zeros((m, 3))
    np.add.at(rsum, inv, colors)
    color = rsum / cnt[:, None]
    coords = unpack(ukeys)
    resid = np.clip(centroid - (coords.astype(np.float64) + 0.5), -0.5, 0.5)
    feats = np.concatenate([centroid / s, color, resid], axis=1)
    order = np.argsort(inv, kind="stable")
    offsets = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    return dict(coords=coords, feats=feats, keys=ukeys, s=s, scale_to_world=1.0 / s,
                point_to_voxel=inv.astype(np.int64), source_order=order.astype(np.int64),
                source_offsets=offsets)


def reconstructed(vox: dict) -> np.ndarray:
    """(coord + 0.5 + residual) * scale (voxelgrid.py:119-122)."""
    return (vox["coords"].astype(np.float64) + 0.5 + vox["feats"][:, 6:9]) * vox["scale_to_world"]


def pool(coords: np.ndarray, feats: np.ndarray, stride: int):
    """Mean of occupied children per stride-doubled parent (voxelgrid.py:171-185)."""
    step = stride * 2
    parents = (coords.astype(np.int64) // step) * step
    ukeys, inv, cnt = np.unique(pack(parents), return_inverse=True, return_counts=True)
    acc = np.zeros((ukeys.size, feats.shape[1]))
    np.add.at(acc, inv, feats)
    return unpack(ukeys), acc / cnt[:, None], ukeys


def tap_offsets(kernel: int) -> np.ndarray:
    """(k^3, 3) (dx, dy, dz) offsets, taps in lexicographic (dz, dy, dx) order
    (sparsenet.py:201-206: tap [a,b,c] is offset (c-r, b-r, a-r))."""
    r = kernel // 2
    a, b, c = np.meshgrid(np.arange(kernel), np.arange(kernel), np.arange(kernel), indexing="ij")
    return np.stack([c.ravel() - r, b.ravel() - r, a.ravel() - r], axis=1).astype(np.int64)


def kernel_map(coords: np.ndarray, keys: np.ndarray, stride: int, kernel: int = 3) -> np.ndarray:
    """(M, k^3) neighbour rows (-1 = empty) for a stride-s conv (sparsenet.py:201-207)."""
    c = coords.astype(np.int64)
    offs = tap_offsets(kernel) * stride
    out = np.empty((c.shape[0], offs.shape[0]), dtype=np.int64)
    for t in range(offs.shape[0]):
        out[:, t] = lookup(keys, c + offs[t])
    return out


def transposed_map(targets: np.ndarray, parent_keys: np.ndarray, parent_stride: int):
    """Parent row (-1 = orphan) and child tap index (dz*4+dy*2+dx) per target
    (sparsenet.py:235-238)."""
    t = targets.astype(np.int64)
    parents = (t // parent_stride) * parent_stride
    d = (t - parents) // (parent_stride // 2)
    tap = d[:, 2] * 4 + d[:, 1] * 2 + d[:, 0]
    return lookup(parent_keys, parents), tap.astype(np.int64)
