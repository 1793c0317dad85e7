"""Adaptive voxelization, voxel hashing and kernel maps on the GPU.

Drop-in for the reference voxelgrid.py (pack_coords 22-27, SparseVoxelGrid
40-94, VoxelizedCloud 97-122, voxelize_adaptive 125-168, pool_2x2x2 171-185);
the work runs in libsfb200 (csrc/voxelize.cu, csrc/hashmap.cu). Results are
bit-identical to the reference: canonical row order, point_to_voxel,
source_order/offsets, float64 features, and every neighbour map.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .gaussians import to_device
from .pcio import DegenerateCloudError, EmptyCloudError, PointCloud

COORD_LIMIT = 1 << 20
_BIAS = 1 << 20


def pack_coords(coords) -> np.ndarray:
    """(M,3) int -> (M,) int64 keys, monotone in (z, y, x) order (host helper)."""
    c = np.asarray(coords, dtype=np.int64)
    if c.size and (np.abs(c) >= COORD_LIMIT).any():
        raise ValueError(f"voxel coordinates must satisfy |c| < {COORD_LIMIT}")
    return ((c[:, 2] + _BIAS) << 42) | ((c[:, 1] + _BIAS) << 21) | (c[:, 0] + _BIAS)


def unpack_coords(keys) -> np.ndarray:
    k = np.asarray(keys, dtype=np.int64)
    mask = (1 << 21) - 1
    return np.stack([(k & mask) - _BIAS, ((k >> 21) & mask) - _BIAS,
                     ((k >> 42) & mask) - _BIAS], axis=1).astype(np.int32)


@dataclass(eq=False)
class SparseVoxelGrid:
    """Device sparse voxel tensor in canonical (packed-key) row order.

    coords (M,3) int32 CUDA, feats (M,C) CUDA (float64 at level 0, float32
    inside the network), stride, scale_to_world. Constructed without ``keys``
    (the reference constructor, voxelgrid.py:57-79), rows are validated and
    sorted by packed key on the device, duplicates rejected; the library's own
    producers (voxelize_adaptive) pass their canonical keys and skip that.
    """

    coords: torch.Tensor
    feats: torch.Tensor
    stride: int = 1
    scale_to_world: float = 1.0
    keys: torch.Tensor = field(default=None, repr=False)

    def __post_init__(self):
        if self.keys is not None:
            return
        c = to_device(self.coords, torch.int32) if not isinstance(self.coords, torch.Tensor) \
            else self.coords.to(device="cuda", dtype=torch.int32)
        f = self.feats
        if not isinstance(f, torch.Tensor):
            f = to_device(np.asarray(f, dtype=np.float64), torch.float64)
        else:
            f = f.to("cuda")
            if not f.is_floating_point():
                f = f.to(torch.float64)
        if f.ndim == 1:                      # scalar channel shorthand
            f = f[:, None]
        if c.ndim != 2 or c.shape[1] != 3:
            raise ValueError(f"coords must be (M, 3), got {tuple(c.shape)}")
        if f.shape[0] != c.shape[0]:
            raise ValueError("feats row count must match coords")
        if self.stride < 1 or (self.stride & (self.stride - 1)) != 0:
            raise ValueError(f"stride must be a power of two, got {self.stride}")
        if self.scale_to_world <= 0:
            raise ValueError("scale_to_world must be positive")
        if c.numel() and bool((c % self.stride != 0).any()):
            raise ValueError(f"all coordinates must be multiples of stride {self.stride}")
        c64 = c.to(torch.int64)
        if c64.numel() and bool((c64.abs() >= COORD_LIMIT).any()):
            raise ValueError(f"voxel coordinates must satisfy |c| < {COORD_LIMIT}")
        keys = ((c64[:, 2] + _BIAS) << 42) | ((c64[:, 1] + _BIAS) << 21) | (c64[:, 0] + _BIAS)
        keys, order = torch.sort(keys, stable=True)
        if keys.numel() > 1 and bool((keys[1:] == keys[:-1]).any()):
            raise ValueError("duplicate voxel coordinates")
        self.coords = c[order].contiguous()
        self.feats = f[order].contiguous()
        self.keys = keys

    def __len__(self) -> int:
        return int(self.coords.shape[0])

    @property
    def channel_count(self) -> int:
        return int(self.feats.shape[1])

    @classmethod
    def from_host(cls, coords, feats, stride=1, scale_to_world=1.0, feat_dtype=torch.float32):
        """Canonicalise like SparseVoxelGrid.__post_init__ (voxelgrid.py:57-79)."""
        coords = np.ascontiguousarray(coords, dtype=np.int32)
        feats = np.asarray(feats, dtype=np.float64)
        if feats.ndim == 1:
            feats = feats[:, None]
        if coords.ndim != 2 or coords.shape[1] != 3:
            raise ValueError(f"coords must be (M, 3), got {coords.shape}")
        if feats.shape[0] != coords.shape[0]:
            raise ValueError("feats row count must match coords")
        if stride < 1 or (stride & (stride - 1)) != 0:
            raise ValueError(f"stride must be a power of two, got {stride}")
        if coords.size and (coords % stride != 0).any():
            raise ValueError(f"all coordinates must be multiples of stride {stride}")
        keys = pack_coords(coords)
        order = np.argsort(keys, kind="stable")
        keys = keys[order]
        if keys.size > 1 and (keys[1:] == keys[:-1]).any():
            raise ValueError("duplicate voxel coordinates")
        return cls(to_device(coords[order], torch.int32), to_device(feats[order], feat_dtype),
                   stride, scale_to_world, to_device(keys, torch.int64))

    def lookup(self, coords) -> torch.Tensor:
        """Row index of each query coordinate, or -1 where unoccupied
        (voxelgrid.py:88-94), int64 on the device; a GPU hash probe."""
        q = coords if isinstance(coords, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(np.atleast_2d(np.asarray(coords, dtype=np.int64))))
        q = q.to("cuda")
        if q.ndim == 1:
            q = q[None, :]
        if q.ndim != 2 or q.shape[1] != 3:
            raise ValueError(f"query coords must be (K, 3), got {tuple(q.shape)}")
        if q.numel() and bool((q.to(torch.int64).abs() >= COORD_LIMIT).any()):
            raise ValueError(f"voxel coordinates must satisfy |c| < {COORD_LIMIT}")
        q = q.to(torch.int32).contiguous()
        nq = int(q.shape[0])
        rows = torch.empty(nq, dtype=torch.int64, device=q.device)
        _lib.context().call("sfb_lookup", _lib.ptr(self.coords), len(self), _lib.ptr(q), nq,
                            _lib.ptr(rows))
        return rows

    def kernel_map(self, kernel: int = 3) -> torch.Tensor:
        """(M, k^3) int32 neighbour rows for a stride-``self.stride`` conv, -1 = empty
        (the tap lookups of sparsenet.py:201-207)."""
        ctx = _lib.context()
        m = len(self)
        out = torch.empty((m, kernel ** 3), dtype=torch.int32, device=self.coords.device)
        ctx.call("sfb_kernel_map", _lib.ptr(self.coords), m, self.stride, kernel, _lib.ptr(out))
        return out


@dataclass(eq=False)
class VoxelizedCloud:
    grid: SparseVoxelGrid
    point_to_voxel: torch.Tensor   # (N,) int32
    source_order: torch.Tensor     # (N,) int32
    source_offsets: torch.Tensor   # (M+1,) int32
    s: float = 0.0
    bbox: tuple = None

    @property
    def source_indices(self) -> list:
        """Per-voxel tensors of contributing original point indices (voxelgrid.py:109-116)."""
        off = self.source_offsets.cpu().tolist()
        return [self.source_order[off[i]:off[i + 1]] for i in range(len(self.grid))]

    def reconstructed_positions(self) -> torch.Tensor:
        g = self.grid
        return (g.coords.to(torch.float64) + 0.5 + g.feats[:, 6:9]) * g.scale_to_world


def device_bbox(positions: torch.Tensor, lane: int = 0) -> np.ndarray:
    """(lo xyz, hi xyz) of device positions via one reduction + 48-byte read-back."""
    n = int(positions.shape[0])
    if n == 0:
        raise EmptyCloudError("empty cloud has no bbox")
    out = np.zeros(6, dtype=np.float64)
    _lib.context(lane=lane).call("sfb_bbox", _lib.ptr(positions), n,
                                 out.ctypes.data_as(_lib.P))
    return out


def lattice_scale(n: int, lo_hi: np.ndarray) -> float:
    """s = (N / V_bbox)^(1/3) with the reference's float64 ops (voxelgrid.py:133-141)."""
    if n < 2:
        raise ValueError("voxelization needs at least 2 points")
    extent = lo_hi[3:6] - lo_hi[0:3]
    volume = float(np.prod(extent))
    if volume <= 0.0:
        raise DegenerateCloudError("bbox volume is zero; cannot pick a density-1 scale")
    return (n / volume) ** (1.0 / 3.0)


def stage_cloud(cloud: PointCloud):
    """Device float64 positions/colors for a cloud (one H2D copy per array if on host)."""
    def dev(a):
        if isinstance(a, torch.Tensor):
            if a.is_cuda:
                return a.contiguous()
            return a.to("cuda", non_blocking=a.is_pinned()).contiguous()
        return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")
    return dev(cloud.positions), dev(cloud.colors)


def voxelize_adaptive(cloud: PointCloud) -> VoxelizedCloud:
    """Density-1 voxelization with centroid merge (voxelgrid.py:125-168), on the GPU."""
    pos, col = stage_cloud(cloud)
    n = int(pos.shape[0])
    if n < 2:
        raise ValueError("voxelization needs at least 2 points")
    lo_hi = device_bbox(pos)
    s = lattice_scale(n, lo_hi)
    dev = pos.device
    coords = torch.empty((n, 3), dtype=torch.int32, device=dev)
    feats = torch.empty((n, 9), dtype=torch.float64, device=dev)
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    p2v = torch.empty(n, dtype=torch.int32, device=dev)
    order = torch.empty(n, dtype=torch.int32, device=dev)
    offsets = torch.empty(n + 1, dtype=torch.int32, device=dev)
    m = _lib.I64(0)
    _lib.context().call("sfb_voxelize", _lib.ptr(pos), _lib.ptr(col), n, s,
                        lo_hi.ctypes.data_as(_lib.P), _lib.ptr(coords), _lib.ptr(feats),
                        _lib.ptr(keys), _lib.ptr(p2v), _lib.ptr(order), _lib.ptr(offsets),
                        _lib.ctypes.byref(m))
    m = m.value
    grid = SparseVoxelGrid(coords[:m], feats[:m], 1, 1.0 / s, keys[:m])
    return VoxelizedCloud(grid, p2v, order, offsets[:m + 1], s, tuple(lo_hi))


def _pool(grid: SparseVoxelGrid):
    m = len(grid)
    c = grid.channel_count
    dev = grid.coords.device
    f64 = grid.feats.dtype == torch.float64
    f = grid.feats.contiguous() if f64 else grid.feats.to(torch.float32).contiguous()
    pc = torch.empty((m, 3), dtype=torch.int32, device=dev)
    pf = torch.empty((m, c), dtype=f.dtype, device=dev)
    c2p = torch.empty(m, dtype=torch.int32, device=dev)
    mp = _lib.I64(0)
    _lib.context().call("sfb_pool_f64" if f64 else "sfb_pool", _lib.ptr(grid.coords), _lib.ptr(f),
                        m, c, grid.stride, _lib.ptr(pc), _lib.ptr(pf), _lib.ptr(c2p),
                        _lib.ctypes.byref(mp))
    mp = mp.value
    parent = SparseVoxelGrid(pc[:mp], pf[:mp], grid.stride * 2, grid.scale_to_world,
                             pack_keys_device(pc[:mp]))
    return parent, c2p


def pack_keys_device(coords: torch.Tensor) -> torch.Tensor:
    """Packed int64 keys of canonical device coords (voxelgrid.py:22-27)."""
    c = coords.to(torch.int64)
    return ((c[:, 2] + _BIAS) << 42) | ((c[:, 1] + _BIAS) << 21) | (c[:, 0] + _BIAS)


def pool_2x2x2(grid: SparseVoxelGrid) -> SparseVoxelGrid:
    """Mean of occupied children per stride-doubled parent (voxelgrid.py:171-185).

    float64 features (the reference's dtype) are pooled in float64 with the
    children summed in child-row order (np.add.at); float32 network features
    stay float32."""
    return _pool(grid)[0]


def pool_with_parents(grid: SparseVoxelGrid):
    """pool_2x2x2 plus the child -> parent row map (used by tests)."""
    return _pool(grid)


def transposed_map(parent: SparseVoxelGrid, targets: torch.Tensor):
    """Parent row (-1 orphan) and child tap of each target (sparsenet.py:233-238)."""
    m = int(targets.shape[0])
    dev = targets.device
    prow = torch.empty(m, dtype=torch.int32, device=dev)
    tap = torch.empty(m, dtype=torch.int32, device=dev)
    _lib.context().call("sfb_transposed_map", _lib.ptr(parent.coords), len(parent), parent.stride,
                        _lib.ptr(targets), m, _lib.ptr(prow), _lib.ptr(tap))
    return prow, tap
