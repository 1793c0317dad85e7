"""GPU voxel hashing / kernel maps / pooling vs the oracle and the reference
goldens: all integer outputs bit-exact, float64 features bit-exact."""
import hashlib

import numpy as np
import pytest
import torch

from oracle import voxel as OV
from paper_2409_16504_b200 import scenes
from paper_2409_16504_b200.pcio import PointCloud
from paper_2409_16504_b200.voxelgrid import (SparseVoxelGrid, pool_with_parents, transposed_map,
                                              voxelize_adaptive)

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def np_(t):
    return t.detach().cpu().numpy()


def check_voxelization(positions, colors):
    got = voxelize_adaptive(PointCloud(positions, colors))
    ref = OV.voxelize(positions, colors)
    assert np.array_equal(np_(got.grid.coords), ref["coords"])
    assert np.array_equal(np_(got.point_to_voxel), ref["point_to_voxel"])
    assert np.array_equal(np_(got.source_order), ref["source_order"])
    assert np.array_equal(np_(got.source_offsets), ref["source_offsets"])
    assert np.array_equal(np_(got.grid.keys), ref["keys"])
    assert np.array_equal(np_(got.grid.feats), ref["feats"]), \
        np.abs(np_(got.grid.feats) - ref["feats"]).max()
    assert got.grid.scale_to_world == ref["scale_to_world"]
    return got, ref


def test_config1_voxelization_matches_reference_golden(golden, c1_arrays):
    cloud, _ = scenes.config1()
    got = voxelize_adaptive(PointCloud(cloud.positions, cloud.colors))
    assert np.array_equal(np_(got.grid.coords), c1_arrays["coords"])
    assert np.array_equal(np_(got.point_to_voxel), c1_arrays["p2v"])
    assert np.array_equal(np_(got.source_order), c1_arrays["source_order"])
    assert np.array_equal(np_(got.source_offsets), c1_arrays["offsets"])
    assert sha(np_(got.grid.feats)) == golden["config1"]["feats"]
    assert got.grid.scale_to_world == golden["config1"]["scale_to_world"]


def test_config1_kernel_maps_and_pooling_bit_exact(c1_arrays):
    for lvl in range(4):
        coords = c1_arrays[f"coords{lvl}"]
        grid = SparseVoxelGrid.from_host(coords, np.zeros((len(coords), 1)), stride=2 ** lvl)
        assert np.array_equal(np_(grid.kernel_map(3)), c1_arrays[f"kmap{lvl}"]), lvl
        if lvl < 3:
            parent, c2p = pool_with_parents(grid)
            assert np.array_equal(np_(parent.coords), c1_arrays[f"coords{lvl + 1}"])
            assert np.array_equal(np_(c2p), c1_arrays[f"tparent{lvl}"])
            prow, tap = transposed_map(parent, grid.coords)
            assert np.array_equal(np_(prow), c1_arrays[f"tparent{lvl}"])
            assert np.array_equal(np_(tap), c1_arrays[f"ttap{lvl}"])


def cube_corners(offset=0.0):
    c = np.stack(np.meshgrid([0.0, 2.0], [0.0, 2.0], [0.0, 2.0], indexing="ij"), -1).reshape(-1, 3)
    return c + offset, np.random.default_rng(0).random((8, 3))


@pytest.mark.parametrize("offset", [0.0, 0.75, 0.3])
def test_cube_corner_cases(offset):
    # voxelgrid tests: s = 1, residual -0.5 / +0.25 per axis (test_voxelgrid.py:81-103)
    got, ref = check_voxelization(*cube_corners(offset))
    assert len(got.grid) == 8


def test_collision_merge_and_duplicates():
    pos = np.array([[0.0, 0.0, 0.0], [2.0, 2.0, 2.0], [1.25, 1.25, 1.25], [1.75, 1.75, 1.75],
                    [0.5, 1.5, 0.5], [1.5, 0.5, 0.5], [0.5, 0.5, 1.5], [1.5, 1.5, 0.25],
                    [1.25, 1.25, 1.25]])
    col = np.random.default_rng(1).random((9, 3))
    got, ref = check_voxelization(pos, col)
    p2v = np_(got.point_to_voxel)
    assert p2v[2] == p2v[3] == p2v[8]


@pytest.mark.parametrize("seed,n,scale", [(4, 1000, 3.0), (5, 50_000, -2.0), (11, 300_000, 1.0)])
def test_random_clouds_including_negative_coords(seed, n, scale):
    rng = np.random.default_rng(seed)
    pos = rng.normal(size=(n, 3)) * scale if scale < 0 else rng.random((n, 3)) * scale
    check_voxelization(pos, rng.random((n, 3)))


def test_degenerate_and_tiny_clouds_raise():
    pos = np.zeros((5, 3))
    pos[:, 0] = np.arange(5)
    with pytest.raises(ValueError):
        voxelize_adaptive(PointCloud(pos, np.zeros((5, 3))))
    with pytest.raises(ValueError):
        voxelize_adaptive(PointCloud(np.zeros((1, 3)), np.zeros((1, 3))))


@pytest.mark.parametrize("kernel,stride", [(1, 1), (3, 1), (5, 1), (3, 2), (3, 4)])
def test_kernel_maps_random_grids(kernel, stride):
    rng = np.random.default_rng(kernel * 10 + stride)
    side = 24
    lattice = np.stack(np.meshgrid(*[np.arange(side)] * 3, indexing="ij"), -1).reshape(-1, 3)
    pick = rng.choice(lattice.shape[0], size=4000, replace=False)
    coords = ((lattice[pick] - 12) * stride).astype(np.int32)
    grid = SparseVoxelGrid.from_host(coords, np.zeros((4000, 1)), stride=stride)
    c = np_(grid.coords)
    ref = OV.kernel_map(c, OV.pack(c), stride, kernel)
    assert np.array_equal(np_(grid.kernel_map(kernel)), ref)


def test_lookup_clipping_at_coordinate_limit():
    lim = (1 << 20) - 1
    coords = np.array([[lim, 0, 0], [lim - 1, 0, 0], [-lim, 5, 5]], dtype=np.int32)
    grid = SparseVoxelGrid.from_host(coords, np.zeros((3, 1)))
    c = np_(grid.coords)
    assert np.array_equal(np_(grid.kernel_map(3)), OV.kernel_map(c, OV.pack(c), 1, 3))
