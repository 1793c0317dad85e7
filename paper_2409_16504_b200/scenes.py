"""Seeded synthetic inputs standing in for the paper's datasets.

None of THuman 2.0 / 8iVFB / BlendedMVS / CWIPC is available, so every
BASELINE.json config is generated here from a fixed recipe: integer voxel
coordinates stored as float64 positions (exactly representable, as from a
10-bit PLY), uint8 colors from a seeded 3-octave value-noise field divided by
255, and pinhole cameras built with ``Camera.look_at`` at a 60 degree
horizontal field of view.

This module only produces host numpy arrays; it is input generation, used by
the tests, ``bench.py`` and the fixture script alike.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

FOV_DEG = 60.0


@dataclass
class Cloud:
    """Plain host cloud: (N,3) float64 positions, (N,3) float64 colors in [0,1]."""

    positions: np.ndarray
    colors: np.ndarray

    def __len__(self) -> int:
        return self.positions.shape[0]


@dataclass
class View:
    """Camera parameters in the reference's convention (p_cam = R p + t)."""

    rotation: np.ndarray
    translation: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int


def value_noise_rgb(pos: np.ndarray, grid: int, seed: int) -> np.ndarray:
    """uint8 colors from a 3-octave trilinear value-noise field.

    Lattice spacings {32,16,8}*(grid/256) with weights {0.5,0.3,0.2}; one
    independent field per channel.
    """
    rng = np.random.default_rng(seed)
    pos = np.asarray(pos, dtype=np.float64)
    acc = np.zeros((pos.shape[0], 3), dtype=np.float64)
    for base, weight in ((32, 0.5), (16, 0.3), (8, 0.2)):
        spacing = base * grid / 256.0
        side = int(math.ceil(grid / spacing)) + 3
        lattice = rng.random((3, side, side, side))
        u = np.clip(pos / spacing, 0.0, side - 2.000001)
        i0 = np.floor(u).astype(np.int64)
        f = u - i0
        for ch in range(3):
            lat = lattice[ch]
            v = np.zeros(pos.shape[0])
            for dz in (0, 1):
                wz = f[:, 2] if dz else 1.0 - f[:, 2]
                for dy in (0, 1):
                    wy = f[:, 1] if dy else 1.0 - f[:, 1]
                    for dx in (0, 1):
                        wx = f[:, 0] if dx else 1.0 - f[:, 0]
                        v += wx * wy * wz * lat[i0[:, 0] + dx, i0[:, 1] + dy, i0[:, 2] + dz]
            acc[:, ch] += weight * v
    return np.clip(np.rint(acc * 255.0), 0, 255).astype(np.uint8)


def _as_cloud(vox: np.ndarray, grid: int, color_seed: int) -> Cloud:
    pos = np.ascontiguousarray(vox, dtype=np.float64)
    rgb = value_noise_rgb(pos, grid, color_seed).astype(np.float64) / 255.0
    return Cloud(pos, np.ascontiguousarray(rgb))


def look_at(eye, target, up, fx, fy, width, height) -> View:
    """Same construction as the reference Camera.look_at (gaussians.py:114-133)."""
    eye = np.asarray(eye, dtype=np.float64)
    z = np.asarray(target, dtype=np.float64) - eye
    z = z / np.linalg.norm(z)
    x = np.cross(np.asarray(up, dtype=np.float64), z)
    x = x / np.linalg.norm(x)
    y = np.cross(z, x)
    rot = np.stack([x, y, z])
    return View(rot, -rot @ eye, float(fx), float(fy), width / 2.0, height / 2.0,
                int(width), int(height))


def _focal(width: int) -> float:
    return (width / 2.0) / math.tan(math.radians(FOV_DEG / 2.0))


def bounding(cloud: Cloud):
    c = cloud.positions.mean(axis=0)
    r = float(np.sqrt(((cloud.positions - c) ** 2).sum(axis=1)).max())
    return c, r


# ---------------------------------------------------------------- config 1
def config1(n_dirs: int = 21_700, seed: int = 0):
    """Sphere r=100 about (128,128,128), surface-sampled on 256^3; one 256^2 view."""
    rng = np.random.default_rng(seed)
    u = rng.normal(size=(n_dirs, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    c = np.array([128.0, 128.0, 128.0])
    vox = np.unique(np.floor(c + 100.0 * u).astype(np.int64), axis=0)
    cloud = _as_cloud(vox, 256, seed + 1)
    eye = c + np.array([0.0, 0.0, -250.0])
    view = look_at(eye, cloud.positions.mean(axis=0), (0.0, 1.0, 0.0),
                   _focal(256), _focal(256), 256, 256)
    return cloud, [view]


# ---------------------------------------------------------------- config 2 / 4
def _ellipsoid_params(seed: int = 0, count: int = 5, grid: int = 1024):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        axes = rng.uniform(40.0, 200.0, size=3)
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        amax = axes.max()
        centre = rng.uniform(amax + 8.0, grid - amax - 8.0, size=3)
        spin_axis = rng.normal(size=3)
        spin_axis /= np.linalg.norm(spin_axis)
        drift = rng.normal(size=3)
        drift /= np.linalg.norm(drift)
        out.append((axes, q, centre, spin_axis, drift))
    return out


def _quat_rot(q):
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


def _axis_angle(axis, angle):
    k = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(angle) * k + (1 - math.cos(angle)) * (k @ k)


def _thomsen_area(a, b, c, p=1.6075):
    return 4.0 * math.pi * (((a * b) ** p + (a * c) ** p + (b * c) ** p) / 3.0) ** (1.0 / p)


# density chosen so the config-2 union lands near 800k unique voxels
C2_DENSITY = 1.35


def ellipsoid_union(frame: int = 0, seed: int = 0, density: float = C2_DENSITY,
                    grid: int = 1024) -> Cloud:
    params = _ellipsoid_params(seed, grid=grid)
    rng = np.random.default_rng(seed if frame == 0 else 1000 + frame)
    pts = []
    for axes, q, centre, spin_axis, drift in params:
        n = int(density * _thomsen_area(*axes))
        d = rng.normal(size=(n, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        local = d * axes
        rot = _quat_rot(q)
        if frame:
            rot = _axis_angle(spin_axis, math.radians(2.0 * frame)) @ rot
        pts.append(local @ rot.T + centre + frame * drift)
    p = np.concatenate(pts)
    p = p + rng.normal(scale=0.5, size=p.shape)
    vox = np.clip(np.floor(p), 0, grid - 1).astype(np.int64)
    return _as_cloud(np.unique(vox, axis=0), grid, seed + 7)


def ring_views(cloud: Cloud, count: int, size: int):
    c, rb = bounding(cloud)
    views = []
    for k in range(count):
        th = 2.0 * math.pi * k / count
        eye = c + 2.5 * rb * np.array([math.sin(th), 0.0, -math.cos(th)])
        views.append(look_at(eye, c, (0.0, 1.0, 0.0), _focal(size), _focal(size), size, size))
    return views


def config2(seed: int = 0, density: float = C2_DENSITY):
    """Union of 5 ellipsoids on 1024^3 (~800k voxels); 8 ring views at 1024^2."""
    cloud = ellipsoid_union(0, seed, density)
    return cloud, ring_views(cloud, 8, 1024)


def config4_frame(frame: int, seed: int = 0, density: float = C2_DENSITY):
    """Frame f of the 64-frame dynamic sequence; one 1024^2 view at theta=2*pi*f/64."""
    cloud = ellipsoid_union(frame, seed, density)
    c, rb = bounding(cloud)
    th = 2.0 * math.pi * frame / 64.0
    eye = c + 2.5 * rb * np.array([math.sin(th), 0.0, -math.cos(th)])
    return cloud, [look_at(eye, c, (0.0, 1.0, 0.0), _focal(1024), _focal(1024), 1024, 1024)]


# ---------------------------------------------------------------- config 3
def config3(seed: int = 0, views: int = 16, size: int = 512):
    """Uniform cube points plus a torus, noisy, 10% dropout, on 512^3; 16 hemisphere views."""
    rng = np.random.default_rng(seed)
    cube = rng.uniform(-1.0, 1.0, size=(100_000, 3))
    th = rng.uniform(0, 2 * math.pi, size=200_000)
    ph = rng.uniform(0, 2 * math.pi, size=200_000)
    torus = np.stack([(0.6 + 0.2 * np.cos(ph)) * np.cos(th),
                      0.2 * np.sin(ph),
                      (0.6 + 0.2 * np.cos(ph)) * np.sin(th)], axis=1)
    p = np.concatenate([cube, torus]) + rng.normal(scale=0.002, size=(300_000, 3))
    p = p[rng.random(p.shape[0]) >= 0.1]
    vox = np.clip(np.floor((p + 1.0) / 2.0 * 512), 0, 511).astype(np.int64)
    cloud = _as_cloud(np.unique(vox, axis=0), 512, seed + 3)
    c, rb = bounding(cloud)
    out = []
    for _ in range(views):
        az = rng.uniform(0, 2 * math.pi)
        el = math.radians(rng.uniform(10.0, 80.0))
        eye = c + 2.5 * rb * np.array([math.cos(el) * math.sin(az), math.sin(el),
                                       -math.cos(el) * math.cos(az)])
        out.append(look_at(eye, c, (0.0, 1.0, 0.0), _focal(size), _focal(size), size, size))
    return cloud, out


# ---------------------------------------------------------------- config 5
def config5(seed: int = 0, views: int = 32, grid: int = 2048):
    """Heightfield terrain plus 50 boxes on 2048^3; 32 ring views at 1920x1080."""
    rng = np.random.default_rng(seed)
    xs = np.arange(grid, dtype=np.float64)
    gx, gz = np.meshgrid(xs, xs, indexing="ij")
    flat = np.stack([gx.ravel(), np.zeros(gx.size), gz.ravel()], axis=1)
    h = value_noise_rgb(flat, grid, seed + 11)[:, 0].astype(np.float64) / 255.0
    height = (300.0 * h + 200.0).astype(np.int64)
    surf = np.stack([gx.ravel().astype(np.int64), height, gz.ravel().astype(np.int64)], axis=1)
    boxes = []
    for _ in range(50):
        ext = rng.integers(10, 121, size=3)
        lo = rng.integers(0, grid - 121, size=3)
        lo[1] = rng.integers(200, 900)
        for axis in range(3):
            for side in (0, ext[axis] - 1):
                a, b = [i for i in range(3) if i != axis]
                ua, ub = np.meshgrid(np.arange(ext[a]), np.arange(ext[b]), indexing="ij")
                face = np.zeros((ua.size, 3), dtype=np.int64)
                face[:, axis] = side
                face[:, a] = ua.ravel()
                face[:, b] = ub.ravel()
                boxes.append(face + lo)
    vox = np.unique(np.concatenate([surf] + boxes), axis=0)
    vox = vox[(vox >= 0).all(axis=1) & (vox < grid).all(axis=1)]
    cloud = _as_cloud(vox, grid, seed + 5)
    c, rb = bounding(cloud)
    out = []
    for k in range(views):
        t = 2.0 * math.pi * k / views
        eye = c + 1.5 * rb * np.array([math.sin(t), 0.35, -math.cos(t)])
        f = 960.0 / math.tan(math.radians(30.0))
        out.append(look_at(eye, c, (0.0, 1.0, 0.0), f, f, 1920, 1080))
    return cloud, out
