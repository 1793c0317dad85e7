"""Point cloud container (reference pcio.py:39-83) with device residency.

Only the in-memory container is on the hot path: float64 positions (N,3) and
colors (N,3) in [0,1]. Host numpy arrays stay on the host until a pipeline
call stages them (pinned, then one H2D copy); torch CUDA tensors are used in
place.
"""
from __future__ import annotations

import numpy as np
import torch


class EmptyCloudError(ValueError):
    """A cloud with zero points where at least one is required."""


class DegenerateCloudError(ValueError):
    """Geometry without the extent an operation needs (e.g. all points coincident)."""


class PointCloud:
    """positions (N,3) float64 world units; colors (N,3) float64 in [0,1];
    normals optional (N,3) unit rows (pcio.py:39-83). Arrays may be host numpy
    or torch tensors (CUDA tensors stay on the device)."""

    def __init__(self, positions, colors, normals=None, validate: bool = True):
        self.positions = _f64(positions)
        self.colors = _f64(colors)
        self.normals = None if normals is None else _f64(normals)
        self._bbox = None
        if self.positions.ndim != 2 or self.positions.shape[1] != 3:
            raise ValueError(f"positions must be (N, 3), got {tuple(self.positions.shape)}")
        if tuple(self.colors.shape) != tuple(self.positions.shape):
            raise ValueError("colors must match positions shape")
        if validate and self.colors.shape[0]:
            lo, hi = float(self.colors.min()), float(self.colors.max())
            if lo < 0.0 or hi > 1.0:
                raise ValueError("color channels must lie in [0, 1]")
        if self.normals is not None:
            if tuple(self.normals.shape) != tuple(self.positions.shape):
                raise ValueError("normals must match positions shape")
            if validate and self.normals.shape[0]:
                if isinstance(self.normals, torch.Tensor):
                    dev = float((self.normals.norm(dim=1) - 1.0).abs().max())
                else:
                    dev = float(np.max(np.abs(np.linalg.norm(self.normals, axis=1) - 1.0)))
                if dev > 1e-6:
                    raise ValueError("normals must be unit length (within 1e-6)")

    def __len__(self) -> int:
        return int(self.positions.shape[0])

    @property
    def bbox(self):
        """(min, max) corners as float64 numpy (3,) arrays; cached after first
        use (pcio.py:73-80). Device clouds reduce on the GPU (sfb_bbox)."""
        if self._bbox is None:
            if len(self) == 0:
                raise EmptyCloudError("empty cloud has no bbox")
            if isinstance(self.positions, torch.Tensor) and self.positions.is_cuda:
                from .voxelgrid import device_bbox
                lo_hi = device_bbox(self.positions)
                self._bbox = (lo_hi[:3].copy(), lo_hi[3:].copy())
            else:
                p = self.positions.numpy() if isinstance(self.positions, torch.Tensor) else self.positions
                self._bbox = (p.min(axis=0), p.max(axis=0))
        return self._bbox

    def with_positions(self, positions) -> "PointCloud":
        """Same colours and normals at new positions (pcio.py:82-83)."""
        return PointCloud(positions, self.colors, self.normals)

    @property
    def on_device(self) -> bool:
        return isinstance(self.positions, torch.Tensor) and self.positions.is_cuda


def _f64(a):
    if isinstance(a, torch.Tensor):
        return a.to(torch.float64).contiguous()
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------- PLY (pcio.py:100-308)
class PlyParseError(ValueError):
    """Malformed PLY header or body; the message names the offending line."""


class PlyUnsupportedError(ValueError):
    """Well-formed PLY that uses a property, type or encoding outside the contract."""


_FLOATS = ("x", "y", "z", "nx", "ny", "nz")
_UCHARS = ("red", "green", "blue")
_FLOAT_TYPES = {"float", "float32"}
_UCHAR_TYPES = {"uchar", "uint8"}


def _header(stream, path: str):
    """(is_binary, vertex_count, property names in order) of a PLY header, with
    the reference's grammar and error classes (pcio.py:124-207)."""
    def line():
        raw = stream.readline()
        if not raw:
            raise PlyParseError(f"{path}: unexpected end of file inside header")
        return raw.decode("ascii", errors="replace").strip()

    first = line()
    if first != "ply":
        raise PlyParseError(f"{path}: first line must be 'ply', got '{first}'")
    is_binary, count, props, in_vertex = None, None, [], False
    while True:
        ln = line()
        if ln == "" or ln.startswith("comment") or ln.startswith("obj_info"):
            continue
        if ln == "end_header":
            break
        f = ln.split()
        if f[0] == "format":
            if len(f) != 3 or f[2] != "1.0":
                raise PlyParseError(f"{path}: bad format line '{ln}'")
            if f[1] == "ascii":
                is_binary = False
            elif f[1] == "binary_little_endian":
                is_binary = True
            elif f[1] == "binary_big_endian":
                raise PlyUnsupportedError(f"{path}: big-endian PLY is not supported")
            else:
                raise PlyParseError(f"{path}: unknown format '{f[1]}'")
        elif f[0] == "element":
            if len(f) != 3:
                raise PlyParseError(f"{path}: bad element line '{ln}'")
            if f[1] != "vertex":
                raise PlyUnsupportedError(f"{path}: only 'vertex' elements are supported, got '{f[1]}'")
            if count is not None:
                raise PlyParseError(f"{path}: duplicate vertex element '{ln}'")
            try:
                count = int(f[2])
            except ValueError:
                raise PlyParseError(f"{path}: bad vertex count in '{ln}'") from None
            in_vertex = True
        elif f[0] == "property":
            if not in_vertex:
                raise PlyParseError(f"{path}: property before any element: '{ln}'")
            if len(f) != 3:
                raise PlyUnsupportedError(f"{path}: unsupported property '{ln}'")
            ptype, name = f[1], f[2]
            if name in _FLOATS:
                if ptype not in _FLOAT_TYPES:
                    raise PlyUnsupportedError(f"{path}: '{name}' must be float32, got {ptype}")
            elif name in _UCHARS:
                if ptype not in _UCHAR_TYPES:
                    raise PlyUnsupportedError(f"{path}: '{name}' must be uchar, got {ptype}")
            else:
                raise PlyUnsupportedError(f"{path}: unsupported property name '{name}'")
            props.append(name)
        else:
            raise PlyParseError(f"{path}: unrecognized header line '{ln}'")
    if is_binary is None:
        raise PlyParseError(f"{path}: missing format line")
    if count is None:
        raise PlyParseError(f"{path}: missing vertex element")
    base = {"x", "y", "z", "red", "green", "blue"}
    got = set(props)
    if len(props) != len(got):
        raise PlyParseError(f"{path}: duplicate vertex property")
    if got != base and got != base | {"nx", "ny", "nz"}:
        raise PlyUnsupportedError(f"{path}: vertex properties must be x y z red green blue"
                                  f" (+ optional nx ny nz); missing {sorted(base - got)}")
    return is_binary, count, props


def load_ply(path, device=None) -> PointCloud:
    """Read an ascii or binary little-endian PLY (pcio.py:210-257) into a
    PointCloud on the GPU. Binary bodies are copied to the device as the
    file's own bytes (15 or 27 per vertex) and decoded there (sfb_ply_decode):
    positions widened from float32, colours / 255, normals renormalised."""
    from . import _lib
    import os
    path = os.fspath(path)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    with open(path, "rb") as fh:
        is_binary, count, props = _header(fh, path)
        if count == 0:
            raise EmptyCloudError(f"{path}: vertex count is zero")
        has_n = "nx" in props
        if is_binary:
            offs, stride = {}, 0
            for p in props:
                offs[p] = stride
                stride += 4 if p in _FLOATS else 1
            raw = fh.read(count * stride)
            if len(raw) < count * stride:
                raise PlyParseError(f"{path}: body truncated, expected {count * stride} bytes")
            body = torch.frombuffer(bytearray(raw), dtype=torch.uint8).pin_memory().to(dev, non_blocking=True)
            pos = torch.empty((count, 3), dtype=torch.float64, device=dev)
            col = torch.empty((count, 3), dtype=torch.float64, device=dev)
            nrm = torch.empty((count, 3), dtype=torch.float64, device=dev) if has_n else None
            layout = (_lib.I32 * 9)(*[offs.get(p, -1) for p in
                                      ("x", "y", "z", "red", "green", "blue", "nx", "ny", "nz")])
            _lib.context(dev.index).call("sfb_ply_decode", _lib.ptr(body), count, stride, layout,
                                         _lib.ptr(pos), _lib.ptr(col), _lib.ptr(nrm))
            return PointCloud(pos, col, nrm, validate=False)
        try:
            rows = np.loadtxt(fh, dtype=np.float64, ndmin=2, max_rows=count)
        except ValueError as exc:
            raise PlyParseError(f"{path}: bad ascii body ({exc})") from None
    if rows.shape[0] < count:
        raise PlyParseError(f"{path}: body has {rows.shape[0]} rows, header says {count}")
    if rows.shape[1] != len(props):
        raise PlyParseError(f"{path}: rows have {rows.shape[1]} values, header declares {len(props)}")
    col_of = {p: rows[:, i] for i, p in enumerate(props)}
    # ascii values round-trip through float32 / uchar exactly like a binary body,
    # then take the same device decode
    rec = np.zeros(count, dtype=np.dtype([(p, "<f4" if p in _FLOATS else "u1") for p in props]))
    for p in props:
        rec[p] = col_of[p]
    tmp = np.frombuffer(rec.tobytes(), dtype=np.uint8)
    stride = rec.dtype.itemsize
    offs = {p: rec.dtype.fields[p][1] for p in props}
    body = torch.from_numpy(tmp.copy()).to(dev)
    pos = torch.empty((count, 3), dtype=torch.float64, device=dev)
    colt = torch.empty((count, 3), dtype=torch.float64, device=dev)
    nrm = torch.empty((count, 3), dtype=torch.float64, device=dev) if has_n else None
    layout = (_lib.I32 * 9)(*[offs.get(p, -1) for p in
                              ("x", "y", "z", "red", "green", "blue", "nx", "ny", "nz")])
    _lib.context(dev.index).call("sfb_ply_decode", _lib.ptr(body), count, stride, layout,
                                 _lib.ptr(pos), _lib.ptr(colt), _lib.ptr(nrm))
    return PointCloud(pos, colt, nrm, validate=False)


def save_ply(cloud: PointCloud, path, binary: bool = True) -> None:
    """Write a PLY load_ply reads back (pcio.py:265-308): float32 positions,
    uchar colours (rint of c*255, clipped), optional float32 normals."""
    import os
    path = os.fspath(path)
    host = lambda a: a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    pos = host(cloud.positions).astype(np.float32)
    rgb = np.clip(np.rint(host(cloud.colors) * 255.0), 0, 255).astype(np.uint8)
    nrm = None if cloud.normals is None else host(cloud.normals).astype(np.float32)
    n = pos.shape[0]
    names = ["x", "y", "z", "red", "green", "blue"] + (["nx", "ny", "nz"] if nrm is not None else [])
    lines = ["ply", "format binary_little_endian 1.0" if binary else "format ascii 1.0",
             f"element vertex {n}"]
    lines += [f"property {'float' if p in _FLOATS else 'uchar'} {p}" for p in names]
    lines.append("end_header")
    rec = np.empty(n, dtype=np.dtype([(p, "<f4" if p in _FLOATS else "u1") for p in names]))
    for a, p in enumerate(("x", "y", "z")):
        rec[p] = pos[:, a]
    for a, p in enumerate(("red", "green", "blue")):
        rec[p] = rgb[:, a]
    if nrm is not None:
        for a, p in enumerate(("nx", "ny", "nz")):
            rec[p] = nrm[:, a]
    try:
        with open(path, "wb") as fh:
            fh.write(("\n".join(lines) + "\n").encode("ascii"))
            if binary:
                fh.write(rec.tobytes())
            else:
                def f32(v):   # shortest decimal that reads back as the same float32
                    return np.format_float_positional(np.float32(v), unique=True, trim="-")
                body = [" ".join(f32(r[p]) if p in _FLOATS else str(int(r[p])) for p in names)
                        for r in rec]
                fh.write(("\n".join(body) + "\n").encode("ascii"))
    except OSError as exc:
        raise OSError(f"cannot write PLY to {path}: {exc}") from exc


class PlyBody:
    """A binary little-endian PLY vertex body kept as the file's own bytes
    (pinned host memory): what a streaming client ships per frame. The fused
    pipeline copies these bytes to the device (15 B per vertex without
    normals, vs 48 B of float64 PointCloud arrays) and decodes them there."""

    ORDER = ("x", "y", "z", "red", "green", "blue", "nx", "ny", "nz")

    def __init__(self, raw: torch.Tensor, count: int, props):
        self.raw, self.count, self.props = raw, int(count), list(props)
        offs, stride = {}, 0
        for p in self.props:
            offs[p] = stride
            stride += 4 if p in _FLOATS else 1
        self.stride = stride
        self.offsets = [offs.get(p, -1) for p in self.ORDER]
        self.has_normals = "nx" in offs

    def __len__(self) -> int:
        return self.count

    @classmethod
    def from_file(cls, path) -> "PlyBody":
        import os
        path = os.fspath(path)
        with open(path, "rb") as fh:
            binary, count, props = _header(fh, path)
            if not binary:
                raise PlyUnsupportedError(f"{path}: PlyBody needs a binary body")
            stride = sum(4 if p in _FLOATS else 1 for p in props)
            raw = fh.read(count * stride)
        if len(raw) < count * stride:
            raise PlyParseError(f"{path}: body truncated, expected {count * stride} bytes")
        return cls(torch.frombuffer(bytearray(raw), dtype=torch.uint8).pin_memory(), count, props)

    @classmethod
    def from_cloud(cls, cloud: PointCloud) -> "PlyBody":
        """The body save_ply(cloud, binary=True) would write, in pinned memory."""
        host = lambda a: a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
        pos = host(cloud.positions).astype(np.float32)
        rgb = np.clip(np.rint(host(cloud.colors) * 255.0), 0, 255).astype(np.uint8)
        props = ["x", "y", "z", "red", "green", "blue"]
        rec = np.empty(pos.shape[0], dtype=np.dtype([(p, "<f4" if p in _FLOATS else "u1") for p in props]))
        for a, p in enumerate(("x", "y", "z")):
            rec[p] = pos[:, a]
        for a, p in enumerate(("red", "green", "blue")):
            rec[p] = rgb[:, a]
        raw = torch.from_numpy(np.frombuffer(rec.tobytes(), dtype=np.uint8).copy()).pin_memory()
        return cls(raw, pos.shape[0], props)
