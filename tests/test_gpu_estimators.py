"""Analytic estimators on the GPU (estimators.py:41-211, _neighbors.py:33-128)
against outputs recorded from the reference (tests/golden/estimators.npz):
kNN bit-exact (indices and squared distances, index tie-breaks included),
global splats exact, local-PCA splats to float64 rounding (covariances
compared through the frame-independent R^T diag(s^2) R)."""
import numpy as np
import pytest
import torch

from conftest import GOLDEN
from paper_2409_16504_b200 import estimators as E
from paper_2409_16504_b200.pcio import PointCloud

pytestmark = pytest.mark.gpu
ARR = dict(np.load(GOLDEN / "estimators.npz"))
NAMES = ("shell", "lattice")


def np_(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("name", NAMES)
def test_knn_bit_exact(name):
    d2, idx = E.nearest_neighbors(ARR[f"{name}_positions"], 16)
    assert np.array_equal(np_(idx), ARR[f"{name}_knn_idx"])
    assert np.array_equal(np_(d2), ARR[f"{name}_knn_d2"])


def cov_of(q, s):
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    r = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                  2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                  2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1).reshape(-1, 3, 3)
    return np.einsum("kji,kj,kjl->kil", r, s * s, r)


@pytest.mark.parametrize("name", NAMES)
def test_local_pca_and_global_vs_reference(name):
    pc = PointCloud(ARR[f"{name}_positions"], ARR[f"{name}_colors"])
    sp = E.estimate_local_pca(pc, E.EstimatorConfig(kind="local_pca"))
    ref = {k: ARR[f"{name}_pca_{k}"] for k in ("scales", "quaternions", "normals", "centers",
                                             "colors", "opacities")}
    np.testing.assert_allclose(np_(sp.scales), ref["scales"], rtol=1e-9, atol=1e-12)
    c_got = cov_of(np_(sp.quaternions), np_(sp.scales))
    c_ref = cov_of(ref["quaternions"], ref["scales"])
    np.testing.assert_allclose(c_got, c_ref, rtol=0, atol=1e-9 * np.abs(c_ref).max())
    # frames (and normals) agree wherever the spectrum is separated
    lam = ref["scales"] ** 2
    sep = (np.diff(np.sort(lam, axis=1), axis=1).min(axis=1) > 1e-6 * lam.max(axis=1))
    qd = np.minimum(np.abs(np_(sp.quaternions) - ref["quaternions"]).max(axis=1),
                    np.abs(np_(sp.quaternions) + ref["quaternions"]).max(axis=1))
    assert (qd[sep] < 1e-7).all(), qd[sep].max()
    assert (np.abs(np_(sp.normals) - ref["normals"]).max(axis=1)[sep] < 1e-7).all()
    assert np.array_equal(np_(sp.centers), ref["centers"]) and np.array_equal(np_(sp.colors), ref["colors"])
    g = E.estimate_global(pc, E.EstimatorConfig(kind="global_isotropic"))
    for k in ("scales", "quaternions", "normals", "opacities"):
        assert np.array_equal(np_(getattr(g, k)), ARR[f"{name}_global_{k}"]), k


def test_run_estimator_routes_and_errors():
    pos = ARR["shell_positions"][:200]
    pc = PointCloud(pos, ARR["shell_colors"][:200])
    for kind in ("global_isotropic", "local_pca", "neural"):
        sp = E.run_estimator(pc, E.EstimatorConfig(kind=kind))
        assert len(sp) == 200
    with pytest.raises(ValueError):
        E.nearest_neighbors(pos[:5], 5)
    with pytest.raises(ValueError):
        E.estimate_local_pca(PointCloud(pos[:10], ARR["shell_colors"][:10]), E.EstimatorConfig())
