"""End-to-end: cloud -> P2ENet -> planes on the GPU vs the CPU oracle end to end,
and the fused frame vs the two-step (estimate_neural, render) path."""
import numpy as np
import pytest
import torch

from oracle import net as ON
from oracle import raster as OR
from paper_2409_16504_b200 import netplan, scenes
from paper_2409_16504_b200.estimators import EstimatorConfig, estimate_neural, run_estimator
from paper_2409_16504_b200.gaussians import Camera
from paper_2409_16504_b200.pcio import PointCloud
from paper_2409_16504_b200.pipeline import render_frame, stats
from paper_2409_16504_b200.rasterizer import render_planes
from conftest import Cam

pytestmark = pytest.mark.gpu
TOL = 2e-3


def np_(t):
    return t.detach().cpu().numpy().astype(np.float64)


@pytest.fixture(scope="module")
def setup():
    cloud, views = scenes.config1()
    w = netplan.init_random(netplan.NetworkPlan(), 0)
    return PointCloud(cloud.positions, cloud.colors), cloud, views[0], w


def test_estimate_neural_params_vs_oracle(setup):
    pc, cloud, view, w = setup
    sp = estimate_neural(pc, w, EstimatorConfig())
    ref = ON.estimate(cloud.positions, cloud.colors, w.as_oracle_layers(), 3)
    scale = ref["vox"]["scale_to_world"]
    d = np_(sp.centers) - ref["centers"]
    assert (np.abs(d) <= 1e-3 * scale).all()
    bound = 1e-3 * np.maximum(np.abs(ref["scales"]), 1e-3 * scale)
    assert (np.abs(np_(sp.scales) - ref["scales"]) <= bound).all()
    for k in ("quaternions", "opacities", "normals"):
        assert np.abs(np_(getattr(sp, k)) - ref[k]).max() <= 1e-3, k
    assert np.array_equal(np_(sp.colors), ref["colors"])


def test_fused_frame_equals_two_step(setup):
    pc, cloud, view, w = setup
    cam = Camera.of(view)
    fused = render_frame(pc, w, cam, ("rgb", "normal", "depth"))
    two = render_planes(estimate_neural(pc, w), cam, ("rgb", "normal", "depth"))
    for k in ("rgb", "normal", "depth", "transmittance"):
        assert torch.equal(getattr(fused, k), getattr(two, k)), k
    st = stats()
    assert st["runs"] <= st["kept"]


def test_end_to_end_vs_cpu_oracle(setup):
    pc, cloud, view, w = setup
    fb = render_frame(pc, w, Camera.of(view), ("rgb", "normal")).numpy()
    est = ON.estimate(cloud.positions, cloud.colors, w.as_oracle_layers(), 3)
    for mode in ("rgb", "normal"):
        ref = OR.render(est, view, mode)
        for plane in (mode, "transmittance"):
            err = np.abs(fb[plane] - ref[plane])
            print(f"e2e {mode}/{plane}: max |d| {err.max():.3g}")
            assert err.max() <= TOL, (mode, plane, err.max())   # every pixel (measured 2.3e-5)


def test_run_estimator_default_weights(setup):
    pc, cloud, view, w = setup
    a = run_estimator(pc, EstimatorConfig(kind="neural"))
    b = estimate_neural(pc, w)
    assert torch.equal(a.centers, b.centers)
    assert len(run_estimator(pc, EstimatorConfig(kind="local_pca"))) == len(pc)


def test_device_resident_inputs(setup):
    pc, cloud, view, w = setup
    dev = PointCloud(torch.from_numpy(cloud.positions).cuda(), torch.from_numpy(cloud.colors).cuda())
    a = render_frame(dev, w, Camera.of(view))
    b = render_frame(pc, w, Camera.of(view))
    assert torch.equal(a.rgb, b.rgb) and torch.equal(a.normal, b.normal)


def test_graph_replay_matches_eager(setup):
    """sfb_frame: eager first call, graph capture on the second, replays after;
    every replay (with a new camera each time) must equal the eager render."""
    from paper_2409_16504_b200 import _lib, scenes as S
    pc, cloud, view, w = setup
    views = S.ring_views(cloud, 4, 128)
    cams = [Camera.of(v) for v in views]
    h, wd = 128, 128
    out = (torch.empty((h, wd, 3), dtype=torch.float32, device="cuda"),
           torch.empty((h, wd, 3), dtype=torch.float32, device="cuda"), None,
           torch.empty((h, wd), dtype=torch.float32, device="cuda"))
    dev = PointCloud(torch.from_numpy(cloud.positions).cuda(), torch.from_numpy(cloud.colors).cuda())
    ctx = _lib.context()
    ctx.lib.sfb_set_graphs(ctx.handle, 0)
    eager = []
    for cam in cams:
        fb = render_frame(dev, w, cam, ("rgb", "normal"))
        eager.append((fb.rgb.clone(), fb.normal.clone(), fb.transmittance.clone()))
    ctx.lib.sfb_set_graphs(ctx.handle, 1)
    for rep in range(2):
        for cam, (r, n, t) in zip(cams, eager):
            render_frame(dev, w, cam, ("rgb", "normal"), out=out)
            torch.cuda.synchronize()
            assert torch.equal(out[0], r) and torch.equal(out[1], n) and torch.equal(out[3], t)


def tie_cloud():
    """Voxels in exact depth ties: s = 1 exactly (N = bbox volume), two points per
    voxel at dyadic offsets (exact centroids, zero residuals), a network whose
    weights are zero (every voxel gets the same head), an axis-aligned camera:
    each z layer of 256 voxels is ONE tie group whose 512 points interleave by
    (shuffled) index in the reference order (rasterizer.py:105)."""
    rng = np.random.default_rng(11)
    i, j, k, u = np.meshgrid(np.arange(16), np.arange(16), np.arange(4), [0.25, 0.75], indexing="ij")
    pts = np.stack([i + u, j + 0.5, k + 0.5], -1).reshape(-1, 3)
    pts = np.concatenate([pts, [[0.0, 0.0, 0.0], [32.03125, 16.0, 4.0]]])
    pts = pts[rng.permutation(pts.shape[0])]
    cols = rng.random(pts.shape)
    plan = netplan.NetworkPlan()
    layers = [(s, np.zeros(s.weight_shape, np.float32), np.zeros(s.out_channels, np.float32))
              for s in plan.layer_specs()]
    head = np.array([0.3, -0.2, 0.1, -0.5, -0.7, -0.3, 0.9, 0.2, -0.1, 0.3, 0.0, 0.2, -0.4, 0.8],
                    np.float32)
    layers[-1] = (layers[-1][0], layers[-1][1], head)
    cam = Cam(np.eye(3), [-8.0, -8.0, 25.0], 60.0, 60.0, 32.0, 32.0, 64, 64)
    return pts, cols, netplan.NetworkWeights(plan, layers), cam


def test_exact_depth_tie_groups():
    pts, cols, w, cam = tie_cloud()
    est = ON.estimate(pts, cols, w.as_oracle_layers(), 3)
    assert est["vox"]["scale_to_world"] == 1.0
    depth = est["centers"][:, 2]
    assert len(np.unique(depth)) <= 6   # the layers tie exactly
    pc = PointCloud(pts, cols)
    gcam = Camera.of(cam)
    fused = render_frame(pc, w, gcam, ("rgb", "normal", "depth"))
    two = render_planes(estimate_neural(pc, w), gcam, ("rgb", "normal", "depth"))
    for k in ("rgb", "normal", "depth", "transmittance"):
        assert torch.equal(getattr(fused, k), getattr(two, k)), k
    got = fused.numpy()
    for mode in ("rgb", "normal", "depth"):
        ref = OR.render(est, cam, mode)
        assert np.abs(got[mode] - ref[mode]).max() <= TOL, mode
        assert np.abs(got["transmittance"] - ref["transmittance"]).max() <= TOL


def test_lanes_and_graphs_bitwise_identical(setup):
    """The same frame through different lanes (own contexts, arenas and graphs)
    and through eager / captured / replayed calls is bitwise identical."""
    pc, cloud, view, w = setup
    cam = Camera.of(view)
    dev = PointCloud(torch.from_numpy(cloud.positions).cuda(), torch.from_numpy(cloud.colors).cuda())
    ref = None
    for lane in (0, 1, 2):
        for _ in range(3):   # eager, capture, replay
            fb = render_frame(dev, w, cam, ("rgb", "normal"), lane=lane)
            torch.cuda.synchronize()
            got = (fb.rgb.clone(), fb.normal.clone(), fb.transmittance.clone())
            if ref is None:
                ref = got
            assert all(torch.equal(a, b) for a, b in zip(got, ref)), lane


def test_fused_frame_edge_cases(setup):
    """Everything culled (camera looking away), tiny clouds, alternating cloud
    sizes on one lane (separate graphs per shape) — all against the two-step path."""
    pc, cloud, view, w = setup
    bg = (0.1, 0.2, 0.3)
    away = Camera(np.diag([-1.0, 1.0, -1.0]) @ Camera.of(view).rotation, Camera.of(view).translation,
                  view.fx, view.fy, view.cx, view.cy, 64, 48)
    away.translation = -away.rotation @ Camera.of(view).eye()
    fb = render_frame(pc, w, away, ("rgb", "normal"), background=bg).numpy()
    assert (fb["transmittance"] == 1.0).all()
    assert np.allclose(fb["rgb"], np.array(bg), atol=1e-7) and (fb["normal"] == 0).all()
    rng = np.random.default_rng(8)
    cam = Camera(np.eye(3), [0.0, 0.0, 5.0], 40.0, 40.0, 16.0, 16.0, 32, 32)
    for n in (2, 3, 17, 2, 17):
        tiny = PointCloud(rng.normal(size=(n, 3)), rng.random((n, 3)))
        a = render_frame(tiny, w, cam, ("rgb", "normal"))
        b = render_planes(estimate_neural(tiny, w), cam, ("rgb", "normal"))
        assert torch.equal(a.rgb, b.rgb) and torch.equal(a.transmittance, b.transmittance), n


def test_staged_pipeline_matches_device(setup):
    """bench.py's e2e pattern: pinned host clouds staged two frames ahead
    (pipeline.stage: uploads + bbox read-back on their own streams), frames
    issued round-robin over lanes, planes read back on per-lane download
    streams — every frame bitwise equal to the device-resident render."""
    from paper_2409_16504_b200.pipeline import stage
    from paper_2409_16504_b200 import scenes as S
    pc, cloud, view, w = setup
    cams = [Camera.of(v) for v in S.ring_views(cloud, 3, 96)]
    host = PointCloud(torch.from_numpy(cloud.positions).pin_memory(),
                      torch.from_numpy(cloud.colors).pin_memory(), validate=False)
    dev = PointCloud(torch.from_numpy(cloud.positions).cuda(), torch.from_numpy(cloud.colors).cuda())
    lanes, n = 3, 9
    streams = [torch.cuda.Stream() for _ in range(lanes)]
    downs = [torch.cuda.Stream() for _ in range(lanes)]
    got = []
    staged = [stage(host, j % lanes) for j in range(2)]
    for i in range(n):
        src = staged.pop(0)
        if i + 2 < n:
            staged.append(stage(host, (i + 2) % lanes))
        lane = i % lanes
        with torch.cuda.stream(streams[lane]):
            fb = render_frame(src, w, cams[i % len(cams)], lane=lane)
            downs[lane].wait_stream(streams[lane])
            with torch.cuda.stream(downs[lane]):
                got.append((fb.rgb.to("cpu", non_blocking=True), fb.normal.to("cpu", non_blocking=True),
                            fb.transmittance.to("cpu", non_blocking=True)))
    torch.cuda.synchronize()
    for i, planes in enumerate(got):
        ref = render_frame(dev, w, cams[i % len(cams)])
        for a, b in zip(planes, (ref.rgb, ref.normal, ref.transmittance)):
            assert torch.equal(a, b.cpu()), i


def test_staging_refuses_to_overwrite_unrendered(setup):
    """A lane has two staging buffers: a third stage() before either staged
    cloud is rendered raises instead of overwriting data a frame will read."""
    from paper_2409_16504_b200.pipeline import stage
    pc, cloud, view, w = setup
    host = PointCloud(torch.from_numpy(cloud.positions).pin_memory(),
                      torch.from_numpy(cloud.colors).pin_memory(), validate=False)
    a, b = stage(host, 5), stage(host, 5)
    with pytest.raises(RuntimeError, match="staging buffers"):
        stage(host, 5)
    cam = Camera.of(view)
    ra = render_frame(a, w, cam, lane=5).rgb.clone()
    rb = render_frame(b, w, cam, lane=5).rgb.clone()
    c = stage(host, 5)   # a buffer is free again
    rc = render_frame(c, w, cam, lane=5).rgb
    torch.cuda.synchronize()
    assert torch.equal(ra, rb) and torch.equal(ra, rc)


def test_tile_list_overflow_falls_back_to_global_list(setup):
    """Fine / super tile lists are sized from the previous frame's demand; a
    frame that needs more renders every run from the global list: same
    planes, bit for bit."""
    from paper_2409_16504_b200 import _lib
    pc, cloud, view, w = setup
    cam = Camera.of(view)
    want = render_frame(pc, w, cam, ("rgb", "normal"))
    ctx = _lib.context()
    ctx.lib.sfb_set_entry_capacity(ctx.handle, 1)
    try:
        got = render_frame(pc, w, cam, ("rgb", "normal"))
        torch.cuda.synchronize()
        st = stats()
    finally:
        ctx.lib.sfb_set_entry_capacity(ctx.handle, 0)
    assert st["fine_entries"] == 0 and st["super_entries"] == 0 and st["global_entries"] == st["runs"]
    for k in ("rgb", "normal", "transmittance"):
        assert torch.equal(getattr(got, k), getattr(want, k)), k
