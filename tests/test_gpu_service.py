"""render_pose on the GPU (service.py:116-136): RGBA8 straight from the
compositor's epilogue, against the frames.json known-answer payloads and the
oracle's quantised planes; the fused cloud -> RGBA8 frame against the two-step
path."""
import hashlib

import numpy as np
import pytest
import torch

from conftest import Cam, kat_cases
from oracle import net as ON
from oracle import raster as OR
from paper_2409_16504_b200 import netplan, scenes, service
from paper_2409_16504_b200.estimators import estimate_neural
from paper_2409_16504_b200.gaussians import Splats
from paper_2409_16504_b200.pcio import PointCloud
from paper_2409_16504_b200.rasterizer import render_planes

pytestmark = pytest.mark.gpu
KEYS = ("centers", "scales", "quaternions", "opacities", "colors", "normals")


def FixedPose(cam, mode, light=None):
    """A pose whose camera is given directly (the KAT records the matrix)."""
    from paper_2409_16504_b200.gaussians import Camera
    return service.CameraPose(Camera.of(cam), mode, light)


def lsb_close(got, want, frac=1e-3):
    diff = np.abs(got.astype(int) - want.astype(int))
    assert diff.max() <= 1 and (diff > 0).mean() < frac, (diff.max(), (diff > 0).mean())
    return int((diff > 0).sum())


def test_frame_kats_render_pose():
    """frames.json payload SHA-256s, rendered by render_pose on the GPU: byte-exact
    (the oracle fallback below only runs to report what differs if that breaks)."""
    arrays, cases = kat_cases()
    sp = Splats(*(arrays[k] for k in KEYS), validate=False)
    exact = 0
    for case in cases:
        cam = Cam(case["rotation"], case["translation"], case["fx"], case["fy"], case["cx"],
                  case["cy"], case["width"], case["height"])
        pose = FixedPose(cam, case["mode"], case.get("light"))
        rgba = service.render_pose(sp, pose, ambient=case["ambient"],
                                   diffuse=case["diffuse"]).cpu().numpy()
        if hashlib.sha256(rgba.tobytes()).hexdigest() == case["payload_sha256"]:
            exact += 1
            continue
        raise AssertionError(f"{case['name']}: RGBA8 payload differs from frames.json")
        ref = OR.render(arrays, cam, "rgb")
        refn = OR.render(arrays, cam, "normal")
        if case["mode"] == "normal":
            want = OR.to_rgba(refn["normal"] * 0.5 + 0.5, refn["transmittance"])
        elif case["mode"] == "relit":
            want = OR.to_rgba(OR.relight(refn["normal"], ref["rgb"], ref["transmittance"],
                                         case["light"], case["ambient"], case["diffuse"]),
                              ref["transmittance"])
        else:
            want = OR.to_rgba(ref["rgb"], ref["transmittance"])
        lsb_close(rgba, want)
    print(f"{exact}/{len(cases)} KAT payloads byte-exact")


@pytest.fixture(scope="module")
def c1():
    cloud, views = scenes.config1()
    w = netplan.init_random(netplan.NetworkPlan(), 0)
    est = ON.estimate(cloud.positions, cloud.colors, w.as_oracle_layers(), 3)
    return cloud, views[0], w, est


@pytest.mark.parametrize("mode", ["rgb", "normal", "relit"])
def test_render_pose_modes_vs_oracle(c1, mode):
    cloud, view, w, est = c1
    sp = Splats(*(est[k] for k in KEYS), validate=False)
    light = (0.0, -0.6, -0.8)
    pose = FixedPose(view, mode, light if mode == "relit" else None)
    got = service.render_pose(sp, pose, background=(0.1, 0.2, 0.3)).cpu().numpy()
    ref = OR.render(est, view, "rgb", background=(0.1, 0.2, 0.3))
    refn = OR.render(est, view, "normal", background=(0.1, 0.2, 0.3))
    if mode == "rgb":
        want = OR.to_rgba(ref["rgb"], ref["transmittance"])
    elif mode == "normal":
        want = OR.to_rgba(refn["normal"] * 0.5 + 0.5, refn["transmittance"])
    else:
        want = OR.to_rgba(OR.relight(refn["normal"], ref["rgb"], ref["transmittance"], light,
                                     0.2, 0.8), ref["transmittance"])
    n = lsb_close(got, want)
    print(f"{mode}: {n} bytes differ by 1 LSB")


@pytest.mark.parametrize("mode", ["rgb", "normal", "relit"])
def test_fused_rgba_frame_equals_two_step(c1, mode):
    cloud, view, w, est = c1
    pc = PointCloud(cloud.positions, cloud.colors)
    pose = FixedPose(view, mode, (0.0, 0.0, -1.0) if mode == "relit" else None)
    fused = service.render_pose_frame(pc, w, pose)
    two = service.render_pose(estimate_neural(pc, w), pose)
    assert torch.equal(fused, two)
    # and the RGBA8 epilogue equals quantising the float planes of one pass
    fb = render_planes(estimate_neural(pc, w), pose.camera(), ("rgb", "normal"))
    if mode == "rgb":
        q = service.to_rgba(fb.rgb, fb.transmittance)
        lsb_close(fused.cpu().numpy(), q.cpu().numpy(), 0.01)


def test_encode_decode_round_trip_device(c1):
    cloud, view, w, est = c1
    pose = service.PoseMessage((1.0, 0.0, 0.0, 0.0), (0.0, 0.0, 400.0), 200.0, 200.0, 64, 48,
                               "rgb", None, 7)
    rgba = service.render_pose(Splats(*(est[k] for k in KEYS), validate=False), pose)
    blob = service.encode_frame(pose, rgba, 123, 456)
    fields, back = service.decode_frame(blob)
    assert fields["sequence"] == 7 and fields["mode"] == "rgb"
    assert np.array_equal(back, rgba.cpu().numpy())


def test_ply_body_frame_equals_cloud_frame(c1):
    """render_pose_frame fed the binary PLY body (decoded on the device) equals
    the float64 cloud's frame: integer positions and uint8/255 colours survive
    the PLY round trip exactly."""
    from paper_2409_16504_b200.pcio import PlyBody
    cloud, view, w, est = c1
    pc = PointCloud(cloud.positions, cloud.colors)
    pose = FixedPose(view, "relit", (0.0, 0.0, -1.0))
    a = service.render_pose_frame(PlyBody.from_cloud(pc), w, pose).clone()
    b = service.render_pose_frame(pc, w, pose)
    assert torch.equal(a, b)
