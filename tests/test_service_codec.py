"""FRM1 codec and pose camera on the host (service.py:139-167, 42-56)."""
import numpy as np
import pytest

from paper_2409_16504_b200 import service


def pose(**kw):
    base = dict(quaternion=(1.0, 0.0, 0.0, 0.0), translation=(0.0, 0.0, 5.0), fx=100.0,
                fy=100.0, width=64, height=48, mode="normal", light_dir=None, sequence=42)
    base.update(kw)
    return service.PoseMessage(**base)


def test_header_layout_and_round_trip():
    p = pose()
    rgba = np.random.default_rng(0).integers(0, 256, size=(48, 64, 4), dtype=np.uint8)
    blob = service.encode_frame(p, rgba, 1000, 2000)
    assert len(blob) == 33 + 64 * 48 * 4 and blob[:4] == b"FRM1"
    fields, back = service.decode_frame(blob)
    assert fields == {"sequence": 42, "width": 64, "height": 48, "mode": "normal",
                      "render_micros": 1000, "preprocess_micros": 2000}
    assert np.array_equal(back, rgba)


def test_codec_errors():
    p = pose()
    with pytest.raises(ValueError):
        service.encode_frame(p, np.zeros((48, 64, 3), np.uint8), 0, 0)
    blob = service.encode_frame(p, np.zeros((48, 64, 4), np.uint8), 0, 0)
    with pytest.raises(ValueError):
        service.decode_frame(blob[:10])
    with pytest.raises(ValueError):
        service.decode_frame(b"XXXX" + blob[4:])
    with pytest.raises(ValueError):
        service.decode_frame(blob[:-1])


def test_pose_camera_is_quaternion_rotation():
    q = np.array([0.9, 0.1, -0.3, 0.2])
    cam = pose(quaternion=tuple(q / np.linalg.norm(q))).camera()
    r = cam.rotation
    assert np.allclose(r @ r.T, np.eye(3)) and np.isclose(np.linalg.det(r), 1.0)
    assert cam.cx == 32.0 and cam.cy == 24.0
