"""render_backward on the GPU (rasterizer.py:229-354, _raster_kernels.py:204-310)
against gradients recorded from the reference (tests/golden/backward.npz) and
against the oracle on the config-1 scene, every mode."""
import numpy as np
import pytest
import torch

from conftest import Cam
from oracle import net as ON
from oracle import raster as OR
from paper_2409_16504_b200 import netplan, scenes
from paper_2409_16504_b200.gaussians import Camera, Splats
from paper_2409_16504_b200.rasterizer import RenderOptions, render_backward

pytestmark = pytest.mark.gpu
KEYS = ("centers", "scales", "quaternions", "opacities", "colors", "normals")
GRADS = ("d_centers", "d_scales", "d_quaternions", "d_opacities", "d_colors", "d_normals")


def close(got, ref, what):
    """Gradient sums run in a different (deterministic) order than the
    reference's sequential pixel loop: relative 1e-8 of the array's scale (depth mode
    sums attributes ~1e2-1e3 with cancellation)."""
    for g in GRADS:
        a = getattr(got, g).detach().cpu().numpy()
        b = ref[g]
        scale = max(np.abs(b).max(), 1e-30)
        err = np.abs(a - b).max()
        assert err <= 1e-8 * scale, f"{what} {g}: max |d| {err:.3g} (scale {scale:.3g})"


def test_backward_matches_reference_golden():
    from conftest import GOLDEN
    arrays = dict(np.load(GOLDEN / "backward.npz"))
    for ci, (seed, n, w, h, term, amax) in enumerate(arrays["cases"]):
        sp = Splats(*(arrays[f"c{ci}_{k}"] for k in KEYS), validate=False)
        cam = Camera(np.eye(3), np.zeros(3), 45.0, 45.0, w / 2.0, h / 2.0, int(w), int(h))
        for mode in ("rgb", "normal", "depth"):
            ref = {g: arrays[f"c{ci}_{mode}_{g}"] for g in GRADS}
            bg = (0.2, 0.4, 0.6) if mode == "rgb" else (0.0, 0.0, 0.0)
            got = render_backward(sp, cam, arrays[f"c{ci}_{mode}_upstream"], mode, bg,
                                  RenderOptions(16, float(amax), bool(term)))
            close(got, ref, f"case {ci} {mode}")


@pytest.fixture(scope="module")
def c1():
    cloud, views = scenes.config1()
    w = netplan.init_random(netplan.NetworkPlan(), 0)
    est = ON.estimate(cloud.positions, cloud.colors, w.as_oracle_layers(), 3)
    return est, views[0]


@pytest.mark.parametrize("mode", ["rgb", "normal", "depth"])
def test_config1_backward_vs_oracle(c1, mode):
    est, view = c1
    rng = np.random.default_rng(3)
    h, w = view.height, view.width
    up = rng.normal(size=(h, w) if mode == "depth" else (h, w, 3))
    bg = (0.3, 0.1, 0.2) if mode == "rgb" else (0.0, 0.0, 0.0)
    sp = Splats(*(est[k] for k in KEYS), validate=False)
    got = render_backward(sp, Camera.of(view), up, mode, bg)
    ref = OR.render_backward(est, view, up, mode, bg)
    close(got, ref, f"config1 {mode}")
    again = render_backward(sp, Camera.of(view), up, mode, bg)
    for g in GRADS:   # deterministic run to run
        assert torch.equal(getattr(got, g), getattr(again, g)), g


def test_backward_culled_and_shape_errors():
    cam = Camera(np.eye(3), np.zeros(3), 40.0, 40.0, 16.0, 16.0, 32, 32)
    sp = Splats([[0, 0, -1.0], [0, 0, 2.0]], [[0.2] * 3] * 2, [[1, 0, 0, 0]] * 2, [0.5, 0.5],
                [[1.0, 0, 0]] * 2, [[0, 0, 1.0]] * 2)
    g = render_backward(sp, cam, np.ones((32, 32, 3)))
    assert float(g.d_centers[0].abs().sum()) == 0.0 and float(g.d_opacities[1].abs()) > 0
    with pytest.raises(ValueError):
        render_backward(sp, cam, np.ones((31, 32, 3)))
