"""The reference's own hot-path unit sweeps, run against the drop-in on the GPU.

Each test restates one reference test (cited file:line under
/root/reference/pkg/tests/) through this package's public API: voxelization
hand cases (test_voxelgrid.py:81-139), sparse conv / transposed conv / UNet /
head cases (test_sparsenet.py:160-436) and blending semantics
(test_rasterizer.py:41-193). Planes are float32 on the device, so exact
reference values are compared after float32 rounding; float64 quantities
(voxel features, head activations) are compared as the reference does.
"""
import numpy as np
import pytest
import torch

from oracle import raster as OR
from paper_2409_16504_b200.gaussians import Camera, Splats
from paper_2409_16504_b200.netplan import ConvLayerSpec, NetworkPlan, NetworkWeights, init_random
from paper_2409_16504_b200.pcio import DegenerateCloudError, EmptyCloudError, PointCloud
from paper_2409_16504_b200.rasterizer import RenderOptions, render
from paper_2409_16504_b200.sparsenet import (HEAD_CHANNELS, activate_head, sparse_conv,
                                              transposed_conv_pruned, unet_forward)
from paper_2409_16504_b200.voxelgrid import (SparseVoxelGrid, VoxelizedCloud, pool_2x2x2,
                                              voxelize_adaptive)

pytestmark = pytest.mark.gpu
EXACT = RenderOptions(alpha_max=1.0, early_termination=False)
NO_TERM = RenderOptions(early_termination=False)


def np_(t):
    return t.detach().cpu().numpy()


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


# ------------------------------------------------------------------ PointCloud / grid API
def test_pointcloud_bbox_with_positions_and_normals():
    rng = np.random.default_rng(0)
    pos = rng.normal(size=(500, 3))
    col = rng.random((500, 3))
    pc = PointCloud(pos, col)
    lo, hi = pc.bbox
    assert np.array_equal(lo, pos.min(axis=0)) and np.array_equal(hi, pos.max(axis=0))
    assert pc.bbox is pc.bbox   # cached (pcio.py:73-80)
    dev = PointCloud(torch.from_numpy(pos).cuda(), torch.from_numpy(col).cuda())
    dlo, dhi = dev.bbox   # device reduction, bit-identical
    assert np.array_equal(dlo, lo) and np.array_equal(dhi, hi)
    moved = pc.with_positions(pos + 1.0)
    assert np.array_equal(moved.colors, col) and np.array_equal(moved.positions, pos + 1.0)
    with pytest.raises(EmptyCloudError):
        PointCloud(np.zeros((0, 3)), np.zeros((0, 3))).bbox
    nrm = rng.normal(size=(500, 3))
    with pytest.raises(ValueError, match="unit length"):
        PointCloud(pos, col, nrm)
    with pytest.raises(ValueError, match="normals must match"):
        PointCloud(pos, col, np.ones((4, 3)))
    unit = nrm / np.linalg.norm(nrm, axis=1, keepdims=True)
    assert PointCloud(pos, col, unit).normals.shape == (500, 3)
    with pytest.raises(ValueError, match="unit length"):
        PointCloud(torch.from_numpy(pos).cuda(), torch.from_numpy(col).cuda(),
                   torch.from_numpy(nrm).cuda())


def test_grid_canonicalises_and_rejects_like_the_reference():
    # voxelgrid.py:57-79: rows sorted by packed key, duplicates / bad stride rejected
    coords = np.array([[1, 0, 0], [0, 0, 1], [0, 1, 0], [0, 0, 0]])
    g = SparseVoxelGrid(coords, np.array([1.0, 2.0, 3.0, 4.0]))
    assert np_(g.coords).tolist() == [[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]]
    assert np_(g.feats)[:, 0].tolist() == [4.0, 1.0, 3.0, 2.0]
    assert g.channel_count == 1
    with pytest.raises(ValueError, match="duplicate"):
        SparseVoxelGrid([[0, 0, 0], [0, 0, 0]], np.zeros(2))
    with pytest.raises(ValueError, match="power of two"):
        SparseVoxelGrid([[0, 0, 0]], np.zeros(1), stride=3)
    with pytest.raises(ValueError, match="multiples"):
        SparseVoxelGrid([[2, 0, 0]], np.zeros(1), stride=4)
    with pytest.raises(ValueError, match="row count"):
        SparseVoxelGrid([[0, 0, 0]], np.zeros(2))
    with pytest.raises(ValueError, match="scale_to_world"):
        SparseVoxelGrid([[0, 0, 0]], np.zeros(1), scale_to_world=0.0)


def test_grid_lookup_matches_searchsorted():
    rng = np.random.default_rng(3)
    lattice = np.stack(np.meshgrid(*[np.arange(-8, 8)] * 3, indexing="ij"), -1).reshape(-1, 3)
    pick = rng.choice(len(lattice), size=1500, replace=False)
    g = SparseVoxelGrid(lattice[pick], rng.normal(size=(1500, 2)))
    q = lattice[rng.integers(0, len(lattice), size=4000)]
    got = np_(g.lookup(q))
    keys = np_(g.keys)
    qk = ((q[:, 2].astype(np.int64) + (1 << 20)) << 42) | ((q[:, 1] + (1 << 20)) << 21) | (q[:, 0] + (1 << 20))
    pos = np.minimum(np.searchsorted(keys, qk), len(keys) - 1)
    want = np.where(keys[pos] == qk, pos, -1)
    assert got.dtype == np.int64 and np.array_equal(got, want)
    assert np_(SparseVoxelGrid(np.zeros((0, 3), int), np.zeros((0, 1))).lookup([[0, 0, 0]])).tolist() == [-1]


def test_pool_2x2x2_float64_means_in_child_order():
    rng = np.random.default_rng(9)
    lattice = np.stack(np.meshgrid(*[np.arange(-6, 6)] * 3, indexing="ij"), -1).reshape(-1, 3)
    pick = rng.choice(len(lattice), size=900, replace=False)
    g = SparseVoxelGrid(lattice[pick], rng.normal(size=(900, 5)))
    p = pool_2x2x2(g)
    # voxelgrid.py:171-185 in numpy
    c = np_(g.coords).astype(np.int64)
    par = (c // 2) * 2
    key = ((par[:, 2] + (1 << 20)) << 42) | ((par[:, 1] + (1 << 20)) << 21) | (par[:, 0] + (1 << 20))
    uniq, inv, cnt = np.unique(key, return_inverse=True, return_counts=True)
    feats = np.zeros((len(uniq), 5))
    np.add.at(feats, inv, np_(g.feats))
    feats /= cnt[:, None]
    assert p.feats.dtype == torch.float64 and p.stride == 2
    assert np.array_equal(np_(p.feats), feats)
    assert np.array_equal(np_(p.keys), uniq)


# ------------------------------------------------------------------ voxelization (test_voxelgrid.py:81-176)
def cube_corner_cloud(offset=0.0):
    c = np.stack(np.meshgrid([0.0, 2.0], [0.0, 2.0], [0.0, 2.0], indexing="ij"), -1).reshape(-1, 3)
    return PointCloud(c + offset, np.random.default_rng(0).random((8, 3)))


def test_cube_corners_hand_computed():
    vox = voxelize_adaptive(cube_corner_cloud())
    g = vox.grid
    assert len(g) == 8 and g.scale_to_world == pytest.approx(1.0)
    np.testing.assert_allclose(np_(g.feats)[:, 6:9], -0.5, atol=1e-12)
    row = int(np_(g.lookup(np.array([[2, 0, 2]])))[0])
    np.testing.assert_allclose(np_(g.feats)[row, 0:3], [2.0, 0.0, 2.0], atol=1e-12)
    vox = voxelize_adaptive(cube_corner_cloud(0.75))
    np.testing.assert_allclose(np_(vox.grid.feats)[:, 6:9], 0.25, atol=1e-12)
    row = int(np_(vox.grid.lookup(np.array([[0, 0, 0]])))[0])
    np.testing.assert_allclose(np_(vox.grid.feats)[row, 0:3], 0.75, atol=1e-12)


def test_collision_merges_centroid_and_mean_color():
    pos = np.array([[0.0, 0.0, 0.0], [2.0, 2.0, 2.0], [1.25, 1.25, 1.25], [1.75, 1.75, 1.75],
                    [0.5, 1.5, 0.5], [1.5, 0.5, 0.5], [0.5, 0.5, 1.5], [1.5, 1.5, 0.25]])
    col = np.zeros((8, 3))
    col[2] = (1.0, 0.0, 0.0)
    col[3] = (0.0, 1.0, 0.0)
    vox = voxelize_adaptive(PointCloud(pos, col))
    row = int(np_(vox.grid.lookup(np.array([[1, 1, 1]])))[0])
    f = np_(vox.grid.feats)[row]
    np.testing.assert_allclose(f[0:3], 1.5, atol=1e-12)
    np.testing.assert_allclose(f[3:6], [0.5, 0.5, 0.0], atol=1e-12)
    np.testing.assert_allclose(f[6:9], 0.0, atol=1e-12)
    assert np_(vox.source_indices[row]).tolist() == [2, 3]
    p2v = np_(vox.point_to_voxel)
    assert p2v[2] == row and p2v[3] == row


def test_duplicate_points_share_a_voxel():
    cloud = cube_corner_cloud()
    vox = voxelize_adaptive(PointCloud(np.vstack([cloud.positions, cloud.positions[0]]),
                                       np.vstack([cloud.colors, cloud.colors[0]])))
    row = int(np_(vox.point_to_voxel)[0])
    assert int(np_(vox.point_to_voxel)[8]) == row
    assert np_(vox.source_indices[row]).tolist() == [0, 8]


def test_uniform_million_occupancy_near_poisson():
    rng = np.random.default_rng(11)
    n = 1_000_000
    vox = voxelize_adaptive(PointCloud(rng.random((n, 3)), np.full((n, 3), 0.5)))
    assert abs(len(vox.grid) / n - 0.632) < 0.02   # 1 - 1/e at density 1


def test_source_arrays_partition_and_reconstruction():
    rng = np.random.default_rng(4)
    cloud = PointCloud(rng.random((1000, 3)) * 3, rng.random((1000, 3)))
    vox = voxelize_adaptive(cloud)
    assert np.array_equal(np.sort(np_(vox.source_order)), np.arange(1000))
    p2v = np_(vox.point_to_voxel)
    for v, rows in enumerate(vox.source_indices):
        assert (p2v[np_(rows)] == v).all()
    rng = np.random.default_rng(5)
    vox = voxelize_adaptive(PointCloud(rng.normal(size=(5000, 3)) * 2, rng.random((5000, 3))))
    np.testing.assert_allclose(np_(vox.reconstructed_positions()), np_(vox.grid.feats)[:, 0:3],
                               atol=1e-5)
    rng = np.random.default_rng(6)
    cloud = PointCloud(rng.random((20000, 3)), rng.random((20000, 3)))
    vox = voxelize_adaptive(cloud)
    recon = np_(vox.reconstructed_positions())[np_(vox.point_to_voxel)]
    err = np.linalg.norm(recon - cloud.positions, axis=1)
    assert err.mean() <= 0.5 * np.sqrt(3.0) * vox.grid.scale_to_world
    vox = voxelize_adaptive(cube_corner_cloud(0.3))
    recon = np_(vox.reconstructed_positions())[np_(vox.point_to_voxel)]
    np.testing.assert_allclose(recon, cube_corner_cloud(0.3).positions, atol=1e-12)
    rng = np.random.default_rng(7)
    r = np_(voxelize_adaptive(PointCloud(rng.random((5000, 3)) * 10 - 5,
                                         rng.random((5000, 3)))).grid.feats)[:, 6:9]
    assert (r >= -0.5).all() and (r <= 0.5).all()


def test_rejects_degenerate_bbox():
    pos = np.zeros((5, 3))
    pos[:, 0] = np.arange(5)   # flat in y and z
    with pytest.raises(DegenerateCloudError):
        voxelize_adaptive(PointCloud(pos, np.zeros((5, 3))))


# ------------------------------------------------------------------ sparse conv (test_sparsenet.py:160-262)
def dense_conv(grid, w, b):
    """Densify, cross-correlate with zero padding, read back at the occupancy."""
    k = w.shape[0]
    r = k // 2
    g = np_(grid.coords).astype(np.int64) // grid.stride
    g = g - g.min(axis=0)
    nx, ny, nz = g.max(axis=0) + 1
    dense = np.zeros((nz + 2 * r, ny + 2 * r, nx + 2 * r, grid.channel_count))
    dense[g[:, 2] + r, g[:, 1] + r, g[:, 0] + r] = np_(grid.feats)
    acc = np.zeros((nz, ny, nx, w.shape[-1])) + b.astype(np.float64)
    for a in range(k):
        for bb in range(k):
            for c in range(k):
                acc += dense[a:a + nz, bb:bb + ny, c:c + nx] @ w[a, bb, c].astype(np.float64)
    return acc[g[:, 2], g[:, 1], g[:, 0]]


def random_grid(rng, max_side=16, channels=4, stride=1, fill=0.3):
    side = int(rng.integers(2, max_side + 1))
    lattice = np.stack(np.meshgrid(*[np.arange(side)] * 3, indexing="ij"), -1).reshape(-1, 3)
    count = max(1, int(fill * len(lattice)))
    pick = rng.choice(len(lattice), size=count, replace=False)
    coords = (lattice[pick] + rng.integers(-3, 3, size=3)) * stride
    return SparseVoxelGrid(coords, rng.normal(size=(count, channels)), stride=stride)


def test_single_voxel_centre_tap_and_orientation():
    rng = np.random.default_rng(1)
    feats = rng.normal(size=(1, 3))
    grid = SparseVoxelGrid([[2, -1, 4]], feats)
    w = rng.normal(size=(3, 3, 3, 3, 2)).astype(np.float32)
    b = rng.normal(size=2).astype(np.float32)
    out = sparse_conv(grid, ConvLayerSpec("conv", 3, 2), w, b)
    want = feats[0].astype(np.float32).astype(np.float64) @ w[1, 1, 1].astype(np.float64) + b
    np.testing.assert_allclose(np_(out.feats)[0], want, rtol=0, atol=1e-5)
    # only the (dz, dy, dx) = (0, 0, +1) tap: each voxel reads its +x neighbour
    grid = SparseVoxelGrid([[0, 0, 0], [1, 0, 0]], np.array([[2.0], [5.0]]))
    w = np.zeros((3, 3, 3, 1, 1), dtype=np.float32)
    w[1, 1, 2, 0, 0] = 1.0
    out = sparse_conv(grid, ConvLayerSpec("conv", 1, 1), w, np.zeros(1, dtype=np.float32))
    ra, rb = np_(out.lookup([[0, 0, 0], [1, 0, 0]]))
    assert np_(out.feats)[ra, 0] == 5.0 and np_(out.feats)[rb, 0] == 0.0


@pytest.mark.parametrize("kernel", [1, 3, 5])
def test_dense_oracle_agreement(kernel):
    rng = np.random.default_rng(kernel)
    for _ in range(6):
        cin, cout = (int(v) for v in rng.integers(1, 7, size=2))
        grid = random_grid(rng, channels=cin)
        spec = ConvLayerSpec("conv", cin, cout, kernel=kernel)
        w = rng.normal(size=spec.weight_shape).astype(np.float32)
        b = rng.normal(size=cout).astype(np.float32)
        out = sparse_conv(grid, spec, w, b)
        assert torch.equal(out.coords, grid.coords)
        np.testing.assert_allclose(np_(out.feats), dense_conv(grid, w, b), rtol=0, atol=1e-4)
    grid = random_grid(rng, max_side=8, channels=3, stride=4)
    spec = ConvLayerSpec("conv", 3, 2)
    w = rng.normal(size=spec.weight_shape).astype(np.float32)
    b = rng.normal(size=2).astype(np.float32)
    np.testing.assert_allclose(np_(sparse_conv(grid, spec, w, b).feats), dense_conv(grid, w, b),
                               rtol=0, atol=1e-4)


def test_relu_channel_mismatch_and_kind():
    grid = SparseVoxelGrid([[0, 0, 0]], np.array([[1.0]]))
    w = np.array([1.0, -1.0], dtype=np.float32).reshape(1, 1, 1, 1, 2)
    out = sparse_conv(grid, ConvLayerSpec("conv", 1, 2, kernel=1), w, np.zeros(2, np.float32), relu=True)
    assert np_(out.feats).tolist() == [[1.0, 0.0]]
    grid = SparseVoxelGrid([[0, 0, 0]], np.ones((1, 2)), stride=2)
    spec = ConvLayerSpec("conv", 3, 2)
    with pytest.raises(ValueError, match="channels"):
        sparse_conv(grid, spec, np.zeros(spec.weight_shape, np.float32), np.zeros(2, np.float32))
    spec = ConvLayerSpec("transposed_conv", 2, 2)
    with pytest.raises(ValueError, match="conv spec"):
        sparse_conv(grid, spec, np.zeros(spec.weight_shape, np.float32), np.zeros(2, np.float32))


def test_transposed_conv_children_orphans_and_targets():
    rng = np.random.default_rng(2)
    feat = rng.normal(size=(1, 3))
    grid = SparseVoxelGrid([[2, -4, 6]], feat, stride=2)
    spec = ConvLayerSpec("transposed_conv", 3, 2)
    w = rng.normal(size=(2, 2, 2, 3, 2)).astype(np.float32)
    b = rng.normal(size=2).astype(np.float32)
    kids = np.array([[2 + dx, -4 + dy, 6 + dz] for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)])
    out = transposed_conv_pruned(grid, spec, w, b, kids)
    assert len(out) == 8 and out.stride == 1
    f0 = feat[0].astype(np.float32).astype(np.float64)
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                row = int(np_(out.lookup([[2 + dx, -4 + dy, 6 + dz]]))[0])
                np.testing.assert_allclose(np_(out.feats)[row], f0 @ w[dz, dy, dx].astype(np.float64) + b,
                                           rtol=0, atol=1e-5)
    grid = SparseVoxelGrid([[0, 0, 0]], np.ones((1, 2)), stride=2)
    spec = ConvLayerSpec("transposed_conv", 2, 2)
    ones = np.ones(spec.weight_shape, dtype=np.float32)
    assert len(transposed_conv_pruned(grid, spec, ones, np.zeros(2, np.float32), np.zeros((0, 3), int))) == 0
    bias = np.array([0.5, -1.5], dtype=np.float32)
    orphan = transposed_conv_pruned(grid, spec, ones, bias, [[4, 0, 0]])
    assert np_(orphan.feats)[0].tolist() == bias.tolist()
    with pytest.raises(ValueError, match="stride"):
        transposed_conv_pruned(SparseVoxelGrid([[0, 0, 0]], np.ones((1, 2))), spec, ones, bias, [[0, 0, 0]])
    with pytest.raises(ValueError, match="multiples"):
        transposed_conv_pruned(SparseVoxelGrid([[0, 0, 0]], np.ones((1, 2)), stride=4), spec, ones,
                               bias, [[1, 0, 0]])
    rng = np.random.default_rng(3)
    for _ in range(8):
        parents = random_grid(rng, max_side=6, channels=2, stride=4)
        kids = (np_(parents.coords)[:, None, :] + 2 * np.array(
            [[dx, dy, dz] for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)])).reshape(-1, 3)
        target = np.unique(kids[rng.random(len(kids)) < 0.4], axis=0)
        spec = ConvLayerSpec("transposed_conv", 2, 3)
        out = transposed_conv_pruned(parents, spec, rng.normal(size=spec.weight_shape).astype(np.float32),
                                     np.zeros(3, np.float32), target)
        assert {tuple(c) for c in np_(out.coords).tolist()} == {tuple(c) for c in target.tolist()}


def random_cloud(rng, n):
    return PointCloud(rng.random((n, 3)) * 4.0, rng.random((n, 3)))


def test_decoder_occupancy_matches_encoder_levels():
    rng = np.random.default_rng(4)
    vox = voxelize_adaptive(random_cloud(rng, 200))
    levels = [vox.grid]
    for _ in range(3):
        levels.append(pool_2x2x2(levels[-1]))
    grid = levels[-1]
    for target in (levels[2], levels[1], levels[0]):
        spec = ConvLayerSpec("transposed_conv", grid.channel_count, 4)
        grid = transposed_conv_pruned(grid, spec, rng.normal(size=spec.weight_shape).astype(np.float32),
                                      np.zeros(4, np.float32), target.coords)
        assert torch.equal(grid.coords, target.coords) and grid.stride == target.stride


# ------------------------------------------------------------------ UNet + head (test_sparsenet.py:319-436)
def identity_vox(grid):
    n = len(grid)
    ar = torch.arange(n, dtype=torch.int32, device="cuda")
    return VoxelizedCloud(grid, ar, ar, torch.arange(n + 1, dtype=torch.int32, device="cuda"))


def test_unet_output_count_and_zero_weights():
    rng = np.random.default_rng(6)
    vox = voxelize_adaptive(random_cloud(rng, 80))
    assert tuple(unet_forward(vox, init_random(NetworkPlan(), 0)).shape) == (80, HEAD_CHANNELS)
    rng = np.random.default_rng(7)
    vox = voxelize_adaptive(random_cloud(rng, 40))
    plan = NetworkPlan()
    layers = [(s, np.zeros(s.weight_shape, np.float32), rng.normal(size=s.out_channels).astype(np.float32))
              for s in plan.layer_specs()]
    raw = np_(unet_forward(vox, NetworkWeights(plan, layers)))
    np.testing.assert_allclose(raw, np.broadcast_to(layers[-1][2], raw.shape), rtol=0, atol=1e-12)
    grid = SparseVoxelGrid([[0, 0, 0], [1, 1, 1]], np.ones((2, 2)))
    with pytest.raises(ValueError, match="plan expects 9"):
        unet_forward(identity_vox(grid), init_random(NetworkPlan(), 0))


def test_translation_equivariance_by_multiples_of_8():
    rng = np.random.default_rng(8)
    vox = voxelize_adaptive(random_cloud(rng, 120))
    w = init_random(NetworkPlan(), 1)
    raw = np_(unet_forward(vox, w))
    shift = torch.tensor([8, -8, 16], dtype=torch.int32, device="cuda")
    moved = VoxelizedCloud(SparseVoxelGrid(vox.grid.coords + shift, vox.grid.feats, vox.grid.stride,
                                           vox.grid.scale_to_world),
                           vox.point_to_voxel, vox.source_order, vox.source_offsets)
    np.testing.assert_allclose(np_(unet_forward(moved, w)), raw, rtol=0, atol=1e-6)


def test_one_level_unet_matches_dense_network():
    rng = np.random.default_rng(9)
    plan = NetworkPlan((9, 4, 6), (4,), 5)
    w = init_random(plan, 2)
    lattice = np.stack(np.meshgrid(*[np.arange(4)] * 3, indexing="ij"), -1).reshape(-1, 3)
    pick = rng.choice(64, size=30, replace=False)
    grid = SparseVoxelGrid(lattice[pick], rng.normal(size=(30, 9)))
    raw = np_(unet_forward(identity_vox(grid), w))
    (s0, w0, b0), (s1, w1, b1), (s2, w2, b2), (_, w3, b3), (_, w4, b4) = w.layers
    f0 = np.maximum(dense_conv(grid, w0, b0), 0.0)
    coords = np_(grid.coords).astype(np.int64)
    parents = {}
    for i, c in enumerate(coords.tolist()):
        parents.setdefault(tuple((np.array(c) // 2) * 2), []).append(i)
    keys = sorted(parents, key=lambda p: (p[2], p[1], p[0]))
    pgrid = SparseVoxelGrid(np.array(keys), np.array([f0[parents[p]].mean(axis=0) for p in keys]),
                            stride=2)
    f1 = np.maximum(dense_conv(pgrid, w1, b1), 0.0)
    pout = {tuple(c): f1[i] for i, c in enumerate(np_(pgrid.coords).tolist())}
    want = np.empty((30, HEAD_CHANNELS))
    for i, c in enumerate(coords):
        tap = c - (c // 2) * 2
        d0 = np.maximum(pout[tuple((c // 2) * 2)] @ w2[tap[2], tap[1], tap[0]].astype(np.float64) + b2, 0.0)
        h = np.maximum(np.concatenate([d0, f0[i]]) @ w3 + b3, 0.0)
        want[i] = h @ w4 + b4
    np.testing.assert_allclose(raw, want, rtol=0, atol=1e-5)


def test_activate_head_sweep_and_fallbacks():
    out = activate_head(np.zeros(14), voxel_scale=0.5)
    assert np_(out.delta).tolist() == [0.0, 0.0, 0.0]
    np.testing.assert_allclose(np_(out.sigma), np.log(2.0) * 0.5, rtol=1e-12, atol=0)
    assert np_(out.quat).tolist() == [1.0, 0.0, 0.0, 0.0] and float(out.opacity) == 0.5
    raw = np.zeros(14)
    raw[10] = 20.0
    assert abs(float(activate_head(raw, 1.0).opacity) - 1.0) < 1e-8
    raw = np.zeros((2, 14))
    raw[0, 11:14] = (1e-9, 0, 0)   # below the 1e-8 cutoff
    raw[1, 11:14] = (2e-8, 0, 0)
    n = np_(activate_head(raw, 1.0).normal)
    assert n[0].tolist() == [0.0, 0.0, 1.0] and n[1].tolist() == [1.0, 0.0, 0.0]
    raw = np.zeros(14)
    raw[6] = -1.0
    assert np_(activate_head(raw, 1.0).quat).tolist() == [1.0, 0.0, 0.0, 0.0]
    raw[3:6] = -1000.0
    assert (np_(activate_head(raw, 2.0).sigma) > 0).all()
    # float64 raw in: inputs below float32 resolution keep their effect
    raw = np.zeros(14)
    raw[0] = 1e-300
    assert float(activate_head(raw, 1.0).delta[0]) == 1e-300
    rng = np.random.default_rng(10)
    raw = rng.normal(scale=2.0, size=(100_000, 14))
    out = activate_head(raw, 0.37)
    assert (np.abs(np_(out.delta)) <= 0.37).all() and (np_(out.sigma) > 0).all()
    np.testing.assert_allclose(np.linalg.norm(np_(out.quat), axis=1), 1.0, rtol=0, atol=1e-12)
    o = np_(out.opacity)
    assert ((o > 0) & (o < 1)).all()
    np.testing.assert_allclose(np.linalg.norm(np_(out.normal), axis=1), 1.0, rtol=0, atol=1e-12)
    with pytest.raises(ValueError, match="14"):
        activate_head(np.zeros(13), 1.0)


# ------------------------------------------------------------------ blending (test_rasterizer.py:41-193)
def axis_camera(width=64, height=64, fx=100.0, fy=100.0):
    return Camera(np.eye(3), np.zeros(3), fx, fy, width / 2.0, height / 2.0, width, height)


def random_scene(rng, n, opacity_range=(0.1, 0.95)):
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    nr = rng.normal(size=(n, 3))
    nr /= np.linalg.norm(nr, axis=1, keepdims=True)
    centers = np.column_stack([rng.uniform(-0.6, 0.6, n), rng.uniform(-0.6, 0.6, n),
                               rng.uniform(2.0, 4.0, n)])
    return dict(centers=centers, scales=rng.uniform(0.03, 0.3, (n, 3)), quaternions=q,
                opacities=rng.uniform(*opacity_range, n), colors=rng.random((n, 3)), normals=nr)


def splats(d):
    return Splats(d["centers"], d["scales"], d["quaternions"], d["opacities"], d["colors"], d["normals"])


def plane(fb, mode):
    return fb.numpy()[mode]


def test_single_opaque_and_coincident_pair_exact_values():
    sp = Splats.single(center=(0, 0, 2), scales=(0.1,) * 3, color=(0.3, 0.6, 0.9))
    fb = render(sp, axis_camera(), "rgb", (1.0, 1.0, 1.0), EXACT).numpy()
    assert fb["rgb"][32, 32].tolist() == f32([0.3, 0.6, 0.9]).tolist()
    assert fb["transmittance"][32, 32] == 0.0
    bg = np.array([1.0, 0.0, 0.0])
    c1, c2 = np.array([1.0, 1.0, 1.0]), np.array([0.0, 1.0, 0.0])
    pair = dict(centers=np.tile([0.0, 0, 2], (2, 1)), scales=np.full((2, 3), 0.1),
                quaternions=np.tile([1.0, 0, 0, 0], (2, 1)), opacities=np.array([0.5, 0.5]),
                colors=np.stack([c1, c2]), normals=np.tile([0.0, 0, 1], (2, 1)))
    got = render(splats(pair), axis_camera(), "rgb", bg, EXACT).numpy()["rgb"][32, 32]
    assert got.tolist() == f32(0.5 * c1 + 0.25 * c2 + 0.25 * bg).tolist()
    pair["colors"] = np.stack([c2, c1])   # identical depths: the lower index is in front
    got = render(splats(pair), axis_camera(), "rgb", bg, EXACT).numpy()["rgb"][32, 32]
    assert got.tolist() == f32(0.5 * c2 + 0.25 * c1 + 0.25 * bg).tolist()


def test_transparent_splat_and_occlusion():
    fb = render(Splats.single(center=(0, 0, 2), opacity=0.0), axis_camera(), "rgb", (0.5, 0.5, 0.5)).numpy()
    assert (fb["rgb"] == 0.5).all() and (fb["transmittance"] == 1.0).all()
    near = dict(centers=[[0, 0, 1.0]], scales=[[2.0] * 3], colors=[[1.0, 0, 0]])
    far = dict(centers=[[0, 0, 3.0]], scales=[[0.2] * 3], colors=[[0, 1.0, 0]])
    both = Splats(np.vstack([far["centers"], near["centers"]]), np.vstack([far["scales"], near["scales"]]),
                  np.tile([1.0, 0, 0, 0], (2, 1)), np.ones(2),
                  np.vstack([far["colors"], near["colors"]]), np.tile([0, 0, 1.0], (2, 1)))
    region = render(both, axis_camera(), "rgb", (0, 0, 0), EXACT).numpy()["rgb"][28:37, 28:37]
    assert region[:, :, 1].max() < 1e-3 and region[:, :, 0].min() > 1.0 - 1e-3


def test_permutation_and_repeat_bitwise():
    rng = np.random.default_rng(0)
    d = random_scene(rng, 40)
    perm = rng.permutation(40)
    a = render(splats(d), axis_camera(), "rgb", (0.1, 0.1, 0.1))
    b = render(splats({k: v[perm] for k, v in d.items()}), axis_camera(), "rgb", (0.1, 0.1, 0.1))
    assert torch.equal(a.rgb, b.rgb) and torch.equal(a.transmittance, b.transmittance)
    d = random_scene(np.random.default_rng(1), 60)
    assert torch.equal(render(splats(d), axis_camera()).rgb, render(splats(d), axis_camera()).rgb)


@pytest.mark.parametrize("mode", ["rgb", "normal", "depth"])
def test_tiled_matches_untiled_reference(mode):
    """render vs render_reference (no tiling, no termination; rasterizer.py:169-206)."""
    rng = np.random.default_rng(42)
    cam = axis_camera(48, 48)
    for _ in range(8):
        d = random_scene(rng, int(rng.integers(1, 80)))
        bg = rng.random(3)
        a = render(splats(d), cam, mode, bg, NO_TERM).numpy()
        b = OR.render_bruteforce(d, cam, mode, bg)
        np.testing.assert_allclose(a[mode], b[mode], rtol=0, atol=1e-6)
        np.testing.assert_allclose(a["transmittance"], b["transmittance"], rtol=0, atol=1e-6)
    d = random_scene(np.random.default_rng(3), 30)
    cam = axis_camera(50, 38)
    a = render(splats(d), cam, "rgb", (0.2, 0.0, 0.7), NO_TERM).numpy()
    b = OR.render_bruteforce(d, cam, "rgb", (0.2, 0.0, 0.7))
    np.testing.assert_allclose(a["rgb"], b["rgb"], rtol=0, atol=1e-6)


def test_partition_of_unity():
    rng = np.random.default_rng(4)
    d = random_scene(rng, 50)
    d["colors"] = np.ones((50, 3))
    fb = render(splats(d), axis_camera(), "rgb", (0, 0, 0), NO_TERM).numpy()
    np.testing.assert_allclose(fb["rgb"][:, :, 0] + fb["transmittance"], 1.0, atol=1e-6)
    d = random_scene(np.random.default_rng(5), 120, opacity_range=(0.7, 1.0))
    d["colors"] = np.ones((120, 3))
    fb = render(splats(d), axis_camera(), "rgb", (0, 0, 0), RenderOptions(early_termination=True)).numpy()
    assert fb["transmittance"].min() < 1.0 / 255.0   # termination fired
    np.testing.assert_allclose(fb["rgb"][:, :, 0] + fb["transmittance"], 1.0, atol=1e-6)


def test_depth_and_normal_planes():
    fb = render(Splats.single(center=(0, 0, 2.5), scales=(0.1,) * 3), axis_camera(), "depth",
                options=EXACT).numpy()
    assert fb["depth"][32, 32] == pytest.approx(2.5, abs=1e-6) and fb["depth"][0, 0] == 0.0
    n1 = np.array([0.0, 0.0, 1.0])
    fb = render(Splats.single(center=(0, 0, 2), scales=(0.1,) * 3, opacity=0.5, normal=tuple(n1)),
                axis_camera(), "normal", (0.7, 0.7, 0.7)).numpy()
    np.testing.assert_allclose(fb["normal"][32, 32], n1, atol=1e-7)
    assert fb["normal"][0, 0].tolist() == [0.0, 0.0, 0.0]
    na, nb = np.array([1.0, 0.0, 0.0]), np.array([0.0, 1.0, 0.0])
    two = Splats(np.array([[0, 0, 2.0], [0, 0, 3.0]]), np.full((2, 3), 0.1), np.tile([1.0, 0, 0, 0], (2, 1)),
                 np.array([0.5, 0.5]), np.full((2, 3), 0.5), np.stack([na, nb]))
    mix = 0.5 * na + 0.25 * nb
    np.testing.assert_allclose(render(two, axis_camera(), "normal", options=EXACT).numpy()["normal"][32, 32],
                               mix / np.linalg.norm(mix), atol=1e-7)


def test_bad_image_and_mode_rejected():
    cam = axis_camera()
    cam.width = 0
    with pytest.raises(ValueError, match="dimensions"):
        render(Splats.single(), cam)
    with pytest.raises(ValueError, match="mode"):
        render(Splats.single(), axis_camera(), "albedo")
