"""Generate the golden fixtures that pin the CPU oracle to the real reference.

Run in the build container only (needs the read-only reference mount):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb \
        python tests/golden/make_golden.py

It imports the reference ``splatforge`` package, runs its hot path on the
config-1 scene (scenes.config1, seed-0 random-init P2ENet), on the render
known-answer scene of ``pkg/tools/make_protocol_fixtures.py`` and on a few
small raster cases, and records exact integer arrays plus SHA-256 digests of
the float64 arrays. Nothing here is hand-written: every value comes out of the
reference. ``tests/test_oracle.py`` replays the oracle against these files.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from splatforge import estimators, rasterizer, service, sparsenet, voxelgrid  # noqa: E402
from splatforge.evalkit import make_scene  # noqa: E402
from splatforge.gaussians import Camera, Splats  # noqa: E402
from splatforge.pcio import PointCloud  # noqa: E402

from paper_2409_16504_b200 import scenes  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def cam_of(v) -> Camera:
    return Camera(v.rotation, v.translation, v.fx, v.fy, v.cx, v.cy, v.width, v.height)


def splat_hashes(sp) -> dict:
    return {k: sha(getattr(sp, k)) for k in
            ("centers", "scales", "quaternions", "opacities", "colors", "normals")}


def config1():
    cloud_np, views = scenes.config1()
    cloud = PointCloud(cloud_np.positions, cloud_np.colors)
    weights = sparsenet.init_random(sparsenet.NetworkPlan(), 0)
    vox = voxelgrid.voxelize_adaptive(cloud)
    g = vox.grid
    arrays = dict(coords=g.coords, p2v=vox.point_to_voxel.astype(np.int32),
                  source_order=vox.source_order.astype(np.int32),
                  offsets=vox.source_offsets.astype(np.int32), feats=g.feats)
    meta = dict(n=len(cloud), m0=len(g), scale_to_world=float(g.scale_to_world),
                positions=sha(cloud.positions), colors=sha(cloud.colors),
                feats=sha(g.feats))
    # encoder grids, kernel maps (27 taps in (dz,dy,dx) order), pooled coords
    grid = g
    levels = []
    for lvl in range(4):
        coords = grid.coords.astype(np.int64)
        kmap = np.empty((len(grid), 27), dtype=np.int32)
        t = 0
        for a in range(3):
            for b in range(3):
                for c in range(3):
                    off = np.array([c - 1, b - 1, a - 1], dtype=np.int64) * grid.stride
                    kmap[:, t] = sparsenet._lookup_clipped(grid, coords + off)
                    t += 1
        arrays[f"kmap{lvl}"] = kmap
        arrays[f"coords{lvl}"] = grid.coords
        levels.append(len(grid))
        if lvl < 3:
            # pool the raw input features: maps depend on coordinates only
            grid = voxelgrid.pool_2x2x2(grid)
    meta["levels"] = levels
    # transposed maps: parent row and child tap of each stride-s target
    for lvl in range(3):
        targets = arrays[f"coords{lvl}"].astype(np.int64)
        ps = 2 ** (lvl + 1)
        parents = (targets // ps) * ps
        pgrid = voxelgrid.SparseVoxelGrid(arrays[f"coords{lvl + 1}"],
                                          np.zeros((levels[lvl + 1], 1)), stride=ps)
        arrays[f"tparent{lvl}"] = sparsenet._lookup_clipped(pgrid, parents).astype(np.int32)
        d = (targets - parents) // (ps // 2)
        arrays[f"ttap{lvl}"] = (d[:, 2] * 4 + d[:, 1] * 2 + d[:, 0]).astype(np.int32)
    raw = sparsenet.unet_forward(vox, weights)
    first = vox.source_order[vox.source_offsets[:-1]]
    arrays["raw_voxel"] = raw[first]
    splats = estimators.estimate_neural(cloud, weights, estimators.EstimatorConfig(kind="neural"))
    meta["splats"] = splat_hashes(splats)
    meta["weights_p2en"] = hashlib.sha256(_p2en_bytes(weights)).hexdigest()
    cam = cam_of(views[0])
    prep = rasterizer._prepare(splats, cam, "rgb", rasterizer.RenderOptions())
    arrays["source"] = prep.source.astype(np.int32)
    arrays["tile_offsets"] = prep.offsets
    meta["ids"] = sha(prep.ids)
    meta["n_ids"] = int(prep.ids.size)
    meta["radius"] = sha(prep.radius)
    meta["sx"] = sha(prep.sx)
    meta["depth"] = sha(prep.depth)
    planes = {}
    for mode in ("rgb", "normal", "depth"):
        fb = rasterizer.render(splats, cam, mode)
        plane = {"rgb": fb.rgb, "normal": fb.normal, "depth": fb.depth}[mode]
        planes[mode] = sha(plane)
        planes[mode + "_T"] = sha(fb.transmittance)
    fb = rasterizer.render(splats, cam, "rgb", background=(0.25, 0.5, 0.75),
                           options=rasterizer.RenderOptions(early_termination=False))
    planes["rgb_bg_noterm"] = sha(fb.rgb)
    meta["planes"] = planes
    np.savez_compressed(OUT / "c1.npz", **arrays)
    return meta


def _p2en_bytes(weights) -> bytes:
    path = Path("/tmp/_golden_w.p2en")
    sparsenet.save_weights(weights, path)
    return path.read_bytes()


def kat():
    """frames.json known-answer renders (pkg/tools/make_protocol_fixtures.py:113-133)."""
    from importlib import util
    spec = util.spec_from_file_location("mpf", REF / "tools" / "make_protocol_fixtures.py")
    mpf = util.module_from_spec(spec)
    spec.loader.exec_module(mpf)
    cloud, _ = make_scene("checker_sphere", 300, seed=1)
    splats = estimators.run_estimator(cloud, estimators.EstimatorConfig(kind="local_pca"))
    frames = json.loads((REF / "frontend" / "fixtures" / "frames.json").read_text())["frames"]
    arrays = dict(centers=splats.centers, scales=splats.scales, quaternions=splats.quaternions,
                  opacities=splats.opacities, colors=splats.colors, normals=splats.normals)
    cases = []
    for (name, message), rec in zip(mpf.FRAME_POSES, frames):
        pose = service.parse_pose(message)
        cam = pose.camera()
        rgba = service.render_pose(splats, pose)
        got = hashlib.sha256(rgba.tobytes()).hexdigest()
        assert got == rec["payload_sha256"], (name, "reference does not reproduce its KAT")
        light = pose.light_dir if pose.light_dir is not None else service._DEFAULT_LIGHT
        cases.append(dict(name=name, mode=pose.mode, rotation=cam.rotation.tolist(),
                          translation=cam.translation.tolist(), fx=cam.fx, fy=cam.fy,
                          cx=cam.cx, cy=cam.cy, width=cam.width, height=cam.height,
                          light=list(light), ambient=service._AMBIENT,
                          diffuse=service._DIFFUSE, payload_sha256=rec["payload_sha256"]))
    np.savez_compressed(OUT / "kat_splats.npz", **arrays)
    return cases


def raster_cases():
    """Small oracle-test scenes from the reference suites, rendered by the reference."""
    out = []
    arrays = {}
    rng = np.random.default_rng(3)
    for i, (n, w, h) in enumerate([(40, 32, 32), (200, 50, 38), (500, 64, 48)]):
        q = rng.normal(size=(n, 4))
        q /= np.linalg.norm(q, axis=1, keepdims=True)
        nr = rng.normal(size=(n, 3))
        nr /= np.linalg.norm(nr, axis=1, keepdims=True)
        sp = Splats(rng.normal(size=(n, 3)) * 0.25 + [0, 0, 2.5], rng.uniform(0.04, 0.2, (n, 3)),
                    q, rng.uniform(0.2, 0.9, n), rng.uniform(0, 1, (n, 3)), nr)
        cam = Camera(np.eye(3), np.zeros(3), 40.0, 40.0, w / 2.0, h / 2.0, w, h)
        rec = dict(seed_index=i, n=n, width=w, height=h, planes={})
        for k in ("centers", "scales", "quaternions", "opacities", "colors", "normals"):
            arrays[f"case{i}_{k}"] = getattr(sp, k)
        for mode in ("rgb", "normal", "depth"):
            fb = rasterizer.render(sp, cam, mode)
            plane = {"rgb": fb.rgb, "normal": fb.normal, "depth": fb.depth}[mode]
            rec["planes"][mode] = sha(plane)
        out.append(rec)
    np.savez_compressed(OUT / "raster_cases.npz", **arrays)
    return out


def main():
    meta = dict(config1=config1(), kat=kat(), raster=raster_cases(),
                generator="tests/golden/make_golden.py",
                reference="/root/reference/pkg/src/splatforge (read-only mount)")
    (OUT / "golden.json").write_text(json.dumps(meta, indent=1))
    print("wrote", OUT / "golden.json")


if __name__ == "__main__":
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")
    main()
