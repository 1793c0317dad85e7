"""Golden gradients of the reference render_backward (rasterizer.py:229-354).

Run in the build container only (needs the read-only reference mount):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb \\
        python tests/golden/make_golden_backward.py

Seeded random splat scenes (generated here, not copied from the reference's
tests), random upstream gradients, every mode and both termination settings;
the gradients come out of the reference itself and are stored as float64
arrays in tests/golden/backward.npz.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from splatforge.gaussians import Camera, Splats  # noqa: E402
from splatforge.rasterizer import RenderOptions, render_backward  # noqa: E402

OUT = Path(__file__).resolve().parent / "backward.npz"
KEYS = ("centers", "scales", "quaternions", "opacities", "colors", "normals")
GRADS = ("d_centers", "d_scales", "d_quaternions", "d_opacities", "d_colors", "d_normals")


def scene(seed: int, n: int):
    rng = np.random.default_rng(seed)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    nr = rng.normal(size=(n, 3))
    nr /= np.linalg.norm(nr, axis=1, keepdims=True)
    return dict(centers=rng.normal(size=(n, 3)) * [0.5, 0.4, 0.3] + [0.0, 0.0, 3.0],
                scales=rng.uniform(0.03, 0.25, (n, 3)), quaternions=q,
                opacities=rng.uniform(0.05, 0.95, n), colors=rng.random((n, 3)), normals=nr)


def main():
    out = {}
    cases = []
    for ci, (seed, n, w, h, term, amax) in enumerate([(1, 120, 48, 40, True, 0.99),
                                                       (2, 200, 50, 38, False, 1.0),
                                                       (3, 80, 32, 32, True, 0.5)]):
        sp = scene(seed, n)
        for k in KEYS:
            out[f"c{ci}_{k}"] = sp[k]
        cam = Camera(np.eye(3), np.zeros(3), 45.0, 45.0, w / 2.0, h / 2.0, w, h)
        rng = np.random.default_rng(100 + seed)
        for mode in ("rgb", "normal", "depth"):
            up = rng.normal(size=(h, w) if mode == "depth" else (h, w, 3))
            bg = (0.2, 0.4, 0.6) if mode == "rgb" else (0.0, 0.0, 0.0)
            g = render_backward(Splats(*(sp[k] for k in KEYS)), cam, up, mode, bg,
                                RenderOptions(16, amax, term))
            out[f"c{ci}_{mode}_upstream"] = up
            for name in GRADS:
                out[f"c{ci}_{mode}_{name}"] = getattr(g, name)
        cases.append([seed, n, w, h, int(term), amax])
    out["cases"] = np.array(cases, dtype=np.float64)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
