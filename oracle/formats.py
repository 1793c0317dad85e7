"""Oracle: PLY body / SPL1 decoding in numpy (TEST INFRASTRUCTURE ONLY, see
oracle/__init__.py). Restates pcio.load_ply's body handling
(pcio.py:210-257: float32 positions widened, uchar colours / 255, normals
renormalised with a (0,0,1) fallback below 1e-12) and gaussians.load_splats
(gaussians.py:292-311). Headers are parsed by the product's host parser."""
from __future__ import annotations

import numpy as np

FLOATS = ("x", "y", "z", "nx", "ny", "nz")


def decode_ply_body(raw: bytes, count: int, props, binary: bool = True):
    if binary:
        dt = np.dtype([(p, "<f4" if p in FLOATS else "u1") for p in props])
        table = np.frombuffer(raw, dtype=dt, count=count)
        col = {p: table[p] for p in props}
    else:
        body = np.loadtxt(raw.decode("ascii").splitlines(), dtype=np.float64, ndmin=2,
                          max_rows=count)
        col = {p: body[:, i] for i, p in enumerate(props)}
        for p in FLOATS:
            if p in col:
                col[p] = col[p].astype(np.float32)
    pos = np.stack([col["x"], col["y"], col["z"]], axis=1).astype(np.float64)
    rgb = np.stack([col["red"], col["green"], col["blue"]], axis=1).astype(np.float64) / 255.0
    nrm = None
    if "nx" in col:
        nrm = np.stack([col["nx"], col["ny"], col["nz"]], axis=1).astype(np.float64)
        norms = np.linalg.norm(nrm, axis=1, keepdims=True)
        fb = norms[:, 0] < 1e-12
        norms[fb] = 1.0
        nrm = nrm / norms
        nrm[fb] = (0.0, 0.0, 1.0)
    return pos, rgb, nrm


def read_ply(path):
    """(positions, colors, normals) of a PLY file via the product header parser."""
    from paper_2409_16504_b200.pcio import _header
    with open(path, "rb") as fh:
        binary, count, props = _header(fh, str(path))
        raw = fh.read()
    return decode_ply_body(raw, count, props, binary)


def decode_spl1(blob: bytes):
    count = int(np.frombuffer(blob[4:8], dtype="<u4")[0])
    rows = np.frombuffer(blob, dtype="<f4", offset=8).reshape(count, 17).astype(np.float64)
    return dict(centers=rows[:, 0:3], scales=rows[:, 3:6], quaternions=rows[:, 6:10],
                opacities=rows[:, 10], colors=rows[:, 11:14], normals=rows[:, 14:17])
