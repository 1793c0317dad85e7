"""The reference's primitive-math sweeps (/root/reference/pkg/tests/test_gaussians.py)
run against the drop-in's device helpers: quaternion <-> rotation (37-74),
covariance assembly (75-115), projection closed forms and culls through the
render path's projection kernel (152-232) and ``eval_alpha`` (234-274).
Expected values are hand-built (angle-axis matrices, f*sigma/z) as in the
reference, and ``project`` is also checked bit-for-bit against the oracle's
restatement of project_kernel on a random batch.
"""
import numpy as np
import pytest

from oracle import raster as OR
from paper_2409_16504_b200.gaussians import (ALPHA_MAX, COV_DILATION, Z_NEAR, Camera, Splats,
                                              assemble_covariance, eval_alpha, project,
                                              quat_to_rotmat, rotmat_to_quat)

pytestmark = pytest.mark.gpu
RZ90 = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])   # R_z(90 deg) by hand


def np_(t):
    return t.detach().cpu().numpy()


def cam64(width=64, height=64, f=100.0):
    return Camera(np.eye(3), np.zeros(3), f, f, width / 2.0, height / 2.0, width, height)


def unit_quats(rng, n):
    q = rng.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def batch(rng, n, z=5.0, smin=0.01, smax=2.0):
    return Splats(rng.normal(size=(n, 3)) + [0.0, 0.0, z], rng.uniform(smin, smax, (n, 3)),
                  unit_quats(rng, n), rng.uniform(0, 1, n), rng.uniform(0, 1, (n, 3)),
                  np.tile([0.0, 0.0, 1.0], (n, 1)))


# ------------------------------------------------------------------ rotations
def test_rotation_closed_forms_and_round_trip():
    np.testing.assert_allclose(np_(quat_to_rotmat([1.0, 0, 0, 0])), np.eye(3))
    h = np.sqrt(0.5)
    np.testing.assert_allclose(np_(quat_to_rotmat([h, 0, 0, h])), RZ90, atol=1e-12)
    r = np_(quat_to_rotmat(unit_quats(np.random.default_rng(0), 200)))
    np.testing.assert_allclose(np.einsum("nij,nkj->nik", r, r), np.broadcast_to(np.eye(3), r.shape),
                               atol=1e-12)
    np.testing.assert_allclose(np.linalg.det(r), 1.0, atol=1e-12)
    # round trip lands on the canonical sign (largest-magnitude component positive)
    q = unit_quats(np.random.default_rng(1), 500)
    lead = np.take_along_axis(q, np.argmax(np.abs(q), axis=1)[:, None], axis=1)
    np.testing.assert_allclose(np_(rotmat_to_quat(quat_to_rotmat(q))), q * np.sign(lead), atol=1e-9)
    for axis in np.eye(3):   # half turns: every extraction branch
        q = np.concatenate([[0.0], axis])
        np.testing.assert_allclose(np_(quat_to_rotmat(rotmat_to_quat(quat_to_rotmat(q)))),
                                   np_(quat_to_rotmat(q)), atol=1e-9)
    with pytest.raises(ValueError, match="zero quaternion"):
        quat_to_rotmat([0.0, 0.0, 0.0, 0.0])


def test_covariance_assembly():
    np.testing.assert_allclose(np_(assemble_covariance([1.0, 0, 0, 0], [2.0, 3.0, 4.0])),
                               np.diag([4.0, 9.0, 16.0]), atol=1e-12)
    h = np.sqrt(0.5)
    cov = np_(assemble_covariance([h, 0, 0, h], [2.0, 1.0, 1.0]))
    np.testing.assert_allclose(cov, RZ90.T @ np.diag([4.0, 1.0, 1.0]) @ RZ90, atol=1e-12)
    np.testing.assert_allclose(cov, np.diag([1.0, 4.0, 1.0]), atol=1e-12)
    rng = np.random.default_rng(2)
    q, s = unit_quats(rng, 100), rng.uniform(0.1, 5.0, (100, 3))
    cov = np_(assemble_covariance(q, s))
    np.testing.assert_allclose(np.linalg.det(cov), np.prod(s * s, axis=1), rtol=1e-9)
    np.testing.assert_allclose(np.linalg.eigvalsh(cov), np.sort(s * s, axis=1), rtol=1e-9)
    np.testing.assert_allclose(cov, np.swapaxes(cov, 1, 2), atol=1e-12)
    q, s = np.array([0.4, -0.3, 0.7, 0.1]), np.array([1.5, 0.7, 2.2])
    assert np.array_equal(np_(assemble_covariance(q, s)), np_(assemble_covariance(-q, s)))
    with pytest.raises(ValueError, match="scales"):
        assemble_covariance([1.0, 0, 0, 0], [1.0, 0.0, 1.0])


# ------------------------------------------------------------------ projection
def test_projection_on_axis_closed_form():
    proj = project(Splats.single(center=(0, 0, 2), scales=(0.5, 0.5, 0.5)), cam64())
    assert len(proj) == 1
    np.testing.assert_allclose(np_(proj.screen_centers)[0], [32.0, 32.0], atol=1e-12)
    # (f sigma / z)^2 = (100 * 0.5 / 2)^2 = 625 on both axes, plus the dilation
    np.testing.assert_allclose(np_(proj.screen_covs)[0], (625.0 + COV_DILATION) * np.eye(2), atol=1e-9)
    assert float(proj.depths[0]) == pytest.approx(2.0)
    assert float(proj.radii[0]) == pytest.approx(3.0 * np.sqrt(625.0 + COV_DILATION))
    for z, sigma in [(2.0, 0.3), (5.0, 1.0), (10.0, 0.05)]:
        cam = cam64(4096, 4096)
        p = project(Splats.single(center=(0, 0, z), scales=(sigma,) * 3), cam)
        std = np.sqrt(float(p.screen_covs[0, 0, 0]) - COV_DILATION)
        assert std == pytest.approx(cam.fx * sigma / z, rel=1e-9)


def test_projection_culls_and_survivor_indices():
    cam = cam64()
    assert len(project(Splats.single(center=(0, 0, -2)), cam)) == 0          # behind
    assert len(project(Splats.single(center=(0, 0, Z_NEAR)), cam)) == 0      # on the near plane
    assert len(project(Splats.single(center=(100.0, 0, 2), scales=(0.01,) * 3), cam)) == 0
    centers = np.array([[0, 0, 2.0], [0, 0, -1.0], [0.1, 0, 3.0]])
    n = len(centers)
    sp = Splats(centers, np.full((n, 3), 0.1), np.tile([1.0, 0, 0, 0], (n, 1)), np.ones(n),
                np.full((n, 3), 0.5), np.tile([0.0, 0, 1.0], (n, 1)))
    p = project(sp, cam)
    assert np_(p.source_index).tolist() == [0, 2]
    np.testing.assert_array_equal(np_(p.colors), np_(sp.colors)[[0, 2]])


def test_projection_positive_definite_and_bitwise_vs_oracle():
    rng = np.random.default_rng(5)
    sp = batch(rng, 300)
    cam = cam64(256, 256)
    p = project(sp, cam)
    assert len(p) > 0
    assert np.linalg.eigvalsh(np_(p.screen_covs)).min() >= COV_DILATION - 1e-9
    # the oracle restates project_kernel (_raster_kernels.py:20-105) in C
    ref = OR.project(np_(sp.centers), np_(sp.quaternions), np_(sp.scales), cam)
    keep = np.flatnonzero(ref["keep"])
    np.testing.assert_array_equal(np_(p.source_index), keep)
    np.testing.assert_array_equal(np_(p.screen_centers), np.stack([ref["sx"], ref["sy"]], 1)[keep])
    np.testing.assert_array_equal(np_(p.depths), ref["depth"][keep])
    np.testing.assert_array_equal(np_(p.radii), ref["radius"][keep])
    np.testing.assert_array_equal(np_(p.screen_covs)[:, 0, 1], ref["b"][keep])


def test_projection_world_rotation_equivariance():
    rng = np.random.default_rng(6)
    spin = np_(quat_to_rotmat(unit_quats(rng, 1)[0]))
    center, quat = np.array([0.4, -0.2, 3.0]), unit_quats(rng, 1)[0]
    scales, normal = np.array([0.5, 1.0, 0.25]), np.array([0.0, 0.6, 0.8])
    cam = cam64()
    base = Splats.single(center=center, scales=scales, quaternion=quat, opacity=0.7,
                         color=(0.2, 0.4, 0.6), normal=normal)
    spun_q = np_(rotmat_to_quat(np_(quat_to_rotmat(quat)) @ spin.T))
    spun = Splats.single(center=spin @ center, scales=scales, quaternion=spun_q, opacity=0.7,
                         color=(0.2, 0.4, 0.6), normal=spin @ normal)
    cam_spun = Camera(cam.rotation @ spin.T, cam.translation, cam.fx, cam.fy, cam.cx, cam.cy,
                      cam.width, cam.height)
    a, b = project(base, cam), project(spun, cam_spun)
    for k in ("screen_centers", "depths", "screen_covs"):
        np.testing.assert_allclose(np_(getattr(a, k)), np_(getattr(b, k)), atol=1e-6)
    np.testing.assert_allclose(np_(b.normals)[0], spin @ normal, atol=1e-12)


# ------------------------------------------------------------------ eval_alpha
def _proj_with(cov, opacity=0.8, center=(32.0, 32.0)):
    import torch
    p = project(Splats.single(center=(0, 0, 2), opacity=opacity), cam64())
    dev = p.screen_covs.device
    p.screen_covs = torch.tensor(np.asarray([cov], dtype=np.float64), device=dev)
    p.screen_centers = torch.tensor([center], dtype=torch.float64, device=dev)
    return p


def test_eval_alpha_closed_forms():
    p = _proj_with(np.eye(2), opacity=0.8)
    assert float(eval_alpha(p, (32.0, 32.0))[0]) == pytest.approx(0.8)
    assert float(eval_alpha(p, (35.0, 32.0))[0]) == pytest.approx(0.8 * np.exp(-4.5), rel=1e-12)
    p = _proj_with(np.eye(2), opacity=1.0)
    assert float(eval_alpha(p, (32.0, 32.0))[0]) == ALPHA_MAX
    assert float(eval_alpha(p, (32.0, 32.0), alpha_max=1.0)[0]) == pytest.approx(1.0)
    p = _proj_with([[4.0, 0.0], [0.0, 1.0]], opacity=1.0, center=(0.0, 0.0))
    assert float(eval_alpha(p, (2.0, 0.0), alpha_max=1.0)[0]) == pytest.approx(np.exp(-0.5))
    assert float(eval_alpha(p, (0.0, 2.0), alpha_max=1.0)[0]) == pytest.approx(np.exp(-2.0))


def test_eval_alpha_monotone_along_rays():
    rng = np.random.default_rng(7)
    p = _proj_with([[4.0, 1.5], [1.5, 2.0]], opacity=0.9)
    for _ in range(20):
        d = rng.normal(size=2)
        d /= np.linalg.norm(d)
        al = [float(eval_alpha(p, np.array([32.0, 32.0]) + t * d)[0]) for t in np.linspace(0, 10, 40)]
        assert all(a >= b - 1e-15 for a, b in zip(al, al[1:]))
