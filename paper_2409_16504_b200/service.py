"""render_pose and the FRM1 frame codec on the GPU (drop-in for the reference
service.py:23-36, 42-56, 116-167; the WebSocket server itself is out of scope).

``render_pose(splats, pose)`` returns the RGBA8 frame of the reference's
``to_rgba(render(...))`` — for ``mode="relit"`` the rgb and normal planes come
from ONE compositing pass and the Lambertian relight + quantisation run in the
compositor's epilogue, so only 4 bytes per pixel leave the kernel.
``render_pose_frame(cloud, weights, pose)`` is the fused streaming path
(cloud -> P2ENet -> RGBA8). Frames are uint8 CUDA tensors (H, W, 4);
``encode_frame`` reads one back and packs the 33-byte FRM1 header.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .gaussians import Camera, Splats
from .netplan import NetworkWeights
from .pcio import PointCloud
from .rasterizer import RenderOptions

FRAME_MAGIC = b"FRM1"
FRAME_HEADER = struct.Struct("<4sIIIBQQ")
MODE_CODES = {"rgb": 0, "normal": 1, "relit": 2}
MODE_NAMES = {code: name for name, code in MODE_CODES.items()}
_AMBIENT = 0.2
_DIFFUSE = 0.8
_DEFAULT_LIGHT = (0.0, 0.0, -1.0)   # headlight for relit poses without one


def quat_to_rotmat(q) -> np.ndarray:
    """Unit-normalised rotation from a (w, x, y, z) quaternion (gaussians.py:160-177)."""
    q = np.asarray(q, dtype=np.float64)
    norm = np.linalg.norm(q)
    if norm < 1e-12:
        raise ValueError("zero quaternion")
    w, x, y, z = q / norm
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


@dataclass(frozen=True)
class PoseMessage:
    """One requested view; quaternion is the camera rotation, wxyz (service.py:42-56)."""

    quaternion: tuple
    translation: tuple
    fx: float
    fy: float
    width: int
    height: int
    mode: str = "rgb"
    light_dir: tuple = None
    sequence: int = 0

    def camera(self) -> Camera:
        return Camera(quat_to_rotmat(self.quaternion), np.asarray(self.translation, np.float64),
                      self.fx, self.fy, self.width / 2.0, self.height / 2.0, self.width, self.height)


@dataclass(frozen=True, eq=False)
class CameraPose:
    """A render_pose request whose camera is given as a Camera (e.g. a ring
    view built with look_at) rather than a quaternion + focal lengths."""

    cam: Camera
    mode: str = "rgb"
    light_dir: tuple = None
    sequence: int = 0

    @property
    def width(self) -> int:
        return int(self.cam.width)

    @property
    def height(self) -> int:
        return int(self.cam.height)

    def camera(self) -> Camera:
        return self.cam


def _shading(mode: str, light_dir, ambient: float, diffuse: float) -> _lib.Shading_t:
    if mode not in MODE_CODES:
        raise ValueError(f"unknown mode {mode!r}; expected one of {tuple(MODE_CODES)}")
    light = np.asarray(_DEFAULT_LIGHT if light_dir is None else light_dir, dtype=np.float64)
    sh = _lib.Shading_t()
    sh.mode = MODE_CODES[mode]
    sh.light[:] = [float(v) for v in light.reshape(3)]
    sh.ambient, sh.diffuse = float(ambient), float(diffuse)
    return sh


def render_pose(splats: Splats, pose: PoseMessage, background=(0.0, 0.0, 0.0),
                options: RenderOptions = None, out: torch.Tensor = None,
                ambient: float = _AMBIENT, diffuse: float = _DIFFUSE) -> torch.Tensor:
    """RGBA8 (H, W, 4) uint8 CUDA tensor of service.render_pose (service.py:123-136)."""
    cam = pose.camera()
    options = options or RenderOptions()
    bg = np.ascontiguousarray(np.asarray(background, dtype=np.float64).reshape(3))
    if out is None:
        out = torch.empty((pose.height, pose.width, 4), dtype=torch.uint8,
                          device=splats.centers.device)
    s, c, o = splats.struct(), cam.struct(), options.struct()
    sh = _shading(pose.mode, pose.light_dir, ambient, diffuse)
    _lib.context().call("sfb_render_rgba", _lib.ctypes.byref(s), _lib.ctypes.byref(c),
                        _lib.ctypes.byref(o), _lib.ctypes.byref(sh), bg.ctypes.data_as(_lib.P),
                        _lib.ptr(out))
    return out


def render_pose_frame(cloud: PointCloud, weights: NetworkWeights, pose: PoseMessage,
                      background=(0.0, 0.0, 0.0), options: RenderOptions = None,
                      out: torch.Tensor = None, lane: int = 0, ambient: float = _AMBIENT,
                      diffuse: float = _DIFFUSE) -> torch.Tensor:
    """Fused cloud -> P2ENet -> RGBA8 frame (the streaming path; CUDA-graph replayed)."""
    from .pipeline import prepare_cloud
    from .sparsenet import ensure_loaded
    ctx = ensure_loaded(weights, lane)
    cam = pose.camera()
    options = options or RenderOptions()
    pos, col, n, s, lo_hi, slot = prepare_cloud(cloud, lane)
    bg = np.ascontiguousarray(np.asarray(background, dtype=np.float64).reshape(3))
    if out is None:
        out = torch.empty((pose.height, pose.width, 4), dtype=torch.uint8, device=pos.device)
    c, o = cam.struct(), options.struct()
    sh = _shading(pose.mode, pose.light_dir, ambient, diffuse)
    try:
        ctx.call("sfb_frame_rgba", _lib.ptr(pos), _lib.ptr(col), n, s, lo_hi.ctypes.data_as(_lib.P),
                 _lib.ctypes.byref(c), _lib.ctypes.byref(o), _lib.ctypes.byref(sh),
                 bg.ctypes.data_as(_lib.P), _lib.ptr(out))
    finally:
        if slot is not None:   # staging buffer free once the enqueued work is done
            slot[2] = torch.cuda.current_stream().record_event()
    return out


def to_rgba(plane: torch.Tensor, transmittance: torch.Tensor) -> torch.Tensor:
    """Quantise a [0,1] plane to RGBA8, alpha = coverage (service.py:116-120)."""
    rgb = torch.clamp(torch.round(plane.to(torch.float64) * 255.0), 0, 255).to(torch.uint8)
    alpha = torch.clamp(torch.round((1.0 - transmittance.to(torch.float64)) * 255.0), 0, 255)
    return torch.cat([rgb, alpha.to(torch.uint8)[:, :, None]], dim=2)


def encode_frame(pose: PoseMessage, rgba, render_micros: int, preprocess_micros: int) -> bytes:
    """33-byte FRM1 header + row-major RGBA8 payload (service.py:139-146)."""
    if isinstance(rgba, torch.Tensor):
        rgba = rgba.detach().cpu().numpy()
    if rgba.shape != (pose.height, pose.width, 4) or rgba.dtype != np.uint8:
        raise ValueError("payload must be (height, width, 4) uint8")
    header = FRAME_HEADER.pack(FRAME_MAGIC, pose.sequence, pose.width, pose.height,
                               MODE_CODES[pose.mode], render_micros, preprocess_micros)
    return header + np.ascontiguousarray(rgba).tobytes()


def decode_frame(blob: bytes):
    """(fields, RGBA array) of a binary frame (service.py:149-167)."""
    if len(blob) < FRAME_HEADER.size:
        raise ValueError(f"frame too short: {len(blob)} bytes")
    magic, sequence, width, height, mode, render_micros, preprocess_micros = \
        FRAME_HEADER.unpack_from(blob)
    if magic != FRAME_MAGIC:
        raise ValueError(f"bad frame magic {magic!r}")
    if mode not in MODE_NAMES:
        raise ValueError(f"unknown mode code {mode}")
    expected = FRAME_HEADER.size + width * height * 4
    if len(blob) != expected:
        raise ValueError(f"expected {expected} bytes, got {len(blob)}")
    rgba = np.frombuffer(blob, dtype=np.uint8, offset=FRAME_HEADER.size)
    fields = {"sequence": sequence, "width": width, "height": height, "mode": MODE_NAMES[mode],
              "render_micros": render_micros, "preprocess_micros": preprocess_micros}
    return fields, rgba.reshape(height, width, 4)
