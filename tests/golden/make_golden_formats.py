"""Golden PLY / SPL1 files and the reference's decode of them (pcio.py:210-308,
gaussians.py:277-311). Build container only:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb \\
        python tests/golden/make_golden_formats.py

A seeded cloud and splat set (generated here) are written with the
reference's own save_ply / save_splats; the files and the SHA-256 of the
reference's load_ply / load_splats outputs go to tests/golden/formats/.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from splatforge.gaussians import Splats, load_splats, save_splats  # noqa: E402
from splatforge.pcio import PointCloud, load_ply, save_ply  # noqa: E402

OUT = Path(__file__).resolve().parent / "formats"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    OUT.mkdir(exist_ok=True)
    rng = np.random.default_rng(21)
    n = 300
    pos = rng.normal(size=(n, 3)) * 37.5
    col = rng.integers(0, 256, size=(n, 3)) / 255.0
    nrm = rng.normal(size=(n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    np.savez_compressed(OUT / "cloud_in.npz", positions=pos, colors=col, normals=nrm)
    meta = {}
    for name, normals, binary in [("bin_normals", nrm, True), ("bin_plain", None, True),
                                  ("ascii_normals", nrm, False)]:
        path = OUT / f"{name}.ply"
        save_ply(PointCloud(pos, col, normals), path, binary=binary)
        c = load_ply(path)
        meta[name] = {"file_sha256": hashlib.sha256(path.read_bytes()).hexdigest(),
                      "positions": sha(c.positions), "colors": sha(c.colors),
                      "normals": None if c.normals is None else sha(c.normals), "n": n}
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    nr = rng.normal(size=(n, 3))
    nr /= np.linalg.norm(nr, axis=1, keepdims=True)
    sp = Splats(rng.normal(size=(n, 3)), rng.uniform(0.01, 2.0, (n, 3)), q, rng.random(n),
                rng.random((n, 3)), nr)
    np.savez_compressed(OUT / "splats_in.npz", centers=sp.centers, scales=sp.scales,
                        quaternions=sp.quaternions, opacities=sp.opacities, colors=sp.colors,
                        normals=sp.normals)
    path = OUT / "splats.spl1"
    save_splats(path, sp)
    back = load_splats(path)
    meta["spl1"] = {"file_sha256": hashlib.sha256(path.read_bytes()).hexdigest(),
                    **{k: sha(getattr(back, k)) for k in ("centers", "scales", "quaternions",
                                                          "opacities", "colors", "normals")}}
    (OUT / "formats.json").write_text(json.dumps(meta, indent=1) + "\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
