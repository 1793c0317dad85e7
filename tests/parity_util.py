"""Full-frame parity of the fused GPU frame against the CPU oracle (test
infrastructure, shared by tests/test_gpu_scale_parity.py and
tools/parity_report.py).

Two comparisons per (cloud, view):

* identical inputs — the GPU's own per-point Gaussians (``estimate_neural``,
  bitwise the geometry the fused frame renders) through the oracle's
  ``_prepare`` (rasterizer.py:99-130) and the CSR-free full-frame oracle
  renderer: the fused frame's rank order must equal the oracle's stable
  argsort of depth (rasterizer.py:105) bit for bit, every rank's tile rect
  the oracle's (_raster_kernels.py:123-130), hence the tile offsets, and the
  planes within 2e-3;
* end to end — GPU cloud -> planes against oracle cloud -> planes (the
  oracle's float64 P2ENet): the planes differ only through the P2ENet
  parameter tolerance (north star: 1e-3 relative).
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import net as ON
from oracle import raster as OR
from oracle import voxel as OV
from paper_2409_16504_b200.estimators import estimate_neural
from paper_2409_16504_b200.gaussians import Camera
from paper_2409_16504_b200.pipeline import render_frame_debug

TOL = 2e-3
KEYS = ("centers", "scales", "quaternions", "opacities", "colors", "normals")
PLANES = ("rgb", "normal", "transmittance")


def np64(t):
    return t.detach().cpu().numpy().astype(np.float64)


def plane_stats(got: dict, ref: dict) -> dict:
    """max |d| and the count of pixels with any channel over 2e-3, per plane."""
    out = {}
    for p in PLANES:
        err = np.abs(got[p] - ref[p])
        if err.ndim == 3:
            err = err.max(axis=2)
        out[p] = {"max_abs": float(err.max()), "over": int((err > TOL).sum())}
    return out


def tile_rects(sx, sy, radius, w, h, tile=16):
    """bin_tiles' clamped tile range per rank (_raster_kernels.py:123-130)."""
    ntx, nty = -(-w // tile), -(-h // tile)
    with np.errstate(invalid="ignore", over="ignore"):
        x0 = np.maximum(np.floor((sx - radius) / tile), 0)
        x1 = np.minimum(np.floor((sx + radius) / tile), ntx - 1)
        y0 = np.maximum(np.floor((sy - radius) / tile), 0)
        y1 = np.minimum(np.floor((sy + radius) / tile), nty - 1)
    return np.stack([x0, x1, y0, y1], axis=1).astype(np.int64)


def tile_offsets(rects, w, h, tile=16):
    """bin_tiles' per-tile counts -> offsets, by 2-D difference arrays."""
    ntx, nty = -(-w // tile), -(-h // tile)
    live = (rects[:, 0] <= rects[:, 1]) & (rects[:, 2] <= rects[:, 3])
    r = rects[live]
    d = np.zeros((nty + 1, ntx + 1), dtype=np.int64)
    np.add.at(d, (r[:, 2], r[:, 0]), 1)
    np.add.at(d, (r[:, 2], r[:, 1] + 1), -1)
    np.add.at(d, (r[:, 3] + 1, r[:, 0]), -1)
    np.add.at(d, (r[:, 3] + 1, r[:, 1] + 1), 1)
    cnt = d.cumsum(0).cumsum(1)[:nty, :ntx].reshape(-1)
    return np.concatenate([[0], np.cumsum(cnt)])


def gpu_splats_np(pc, weights) -> dict:
    sp = estimate_neural(pc, weights)
    return {k: np64(getattr(sp, k)) for k in KEYS}


def order_parity(dbg: dict, sp: dict, view) -> dict:
    """Fused-frame rank order and run rects vs the oracle's _prepare on the
    same (GPU) Gaussians."""
    w, h = int(view.width), int(view.height)
    prep = OR.prepare(sp, view, "rgb", 16, ty_window=(0, 0))   # sort + support radius only
    src = dbg["source"].cpu().numpy()
    ref_src = prep["source"]
    same_len = src.size == ref_src.size
    mism = int((src != ref_src).sum()) if same_len else -1
    start = dbg["run_start"].cpu().numpy().astype(np.int64)
    count = dbg["run_count"].cpu().numpy().astype(np.int64)
    rect = dbg["run_rect"].cpu().numpy().astype(np.int64)
    o = np.argsort(start, kind="stable")
    start, count, rect = start[o], count[o], rect[o]
    contiguous = bool(start.size and start[0] == 0 and (start[1:] == start[:-1] + count[:-1]).all()
                      and start[-1] + count[-1] == src.size)
    per_rank = np.repeat(rect, count, axis=0)
    want = tile_rects(prep["sx"], prep["sy"], prep["radius"], w, h)
    empty_g = (per_rank[:, 0] > per_rank[:, 1]) | (per_rank[:, 2] > per_rank[:, 3])
    empty_w = (want[:, 0] > want[:, 1]) | (want[:, 2] > want[:, 3])
    rect_ok = per_rank.shape == want.shape and bool(
        (empty_g == empty_w).all() and (per_rank[~empty_g] == want[~empty_w]).all())
    off_g = tile_offsets(per_rank, w, h)
    off_w = tile_offsets(want, w, h)
    return {"kept": int(src.size), "ranks_mismatched": mism, "order_exact": same_len and mism == 0,
            "runs": int(count.size), "runs_contiguous": contiguous, "rects_exact": rect_ok,
            "offsets_exact": bool(np.array_equal(off_g, off_w)), "entries": int(off_w[-1])}


def level_parity(dbg: dict, vox_coords: np.ndarray) -> dict:
    """Fused UNet levels (rows in the path's own order) vs the oracle's
    canonical pooling and 27-tap kernel maps, compared through coordinates."""
    res = []
    coords = vox_coords.astype(np.int64)
    feats = np.zeros((coords.shape[0], 1))
    keys = OV.pack(coords)
    stride = 1
    for lvl, (gc, gm) in enumerate(zip(dbg["level_coords"], dbg["level_maps"])):
        gc = gc.cpu().numpy().astype(np.int64)
        gm = gm.cpu().numpy()
        ok_set = gc.shape == coords.shape and np.array_equal(np.sort(OV.pack(gc)), keys)
        ok_map = False
        if ok_set:
            perm = OV.lookup(keys, gc)               # fused row -> canonical row
            ref = OV.kernel_map(coords, keys, stride)   # (m, 27) canonical
            want = ref[perm]                             # canonical neighbour of each fused row
            got = np.where(gm.T >= 0, perm[np.maximum(gm.T, 0)], -1)
            ok_map = bool(np.array_equal(got, want))
        res.append({"level": lvl, "voxels": int(gc.shape[0]), "coords_exact": bool(ok_set),
                    "map_exact": ok_map})
        if lvl + 1 < len(dbg["level_coords"]):
            coords, feats, keys = OV.pool(coords, feats, stride)
            coords = coords.astype(np.int64)
            stride *= 2
    return {"levels": res, "exact": all(r["coords_exact"] and r["map_exact"] for r in res)}


def frame_parity(pc, cloud, weights, view, est=None, gpu_sp=None, levels=True) -> dict:
    """Every comparison for one (cloud, view); ``est`` = oracle estimate
    (ON.estimate), ``gpu_sp`` = the GPU per-point Gaussians (numpy)."""
    cam = Camera.of(view)
    fb, dbg = render_frame_debug(pc, weights, cam, ("rgb", "normal"))
    got = fb.numpy()
    if gpu_sp is None:
        gpu_sp = gpu_splats_np(pc, weights)
    rec = {"order": order_parity(dbg, gpu_sp, view)}
    same = OR.render_stream(gpu_sp, view, ("rgb", "normal"))
    rec["renderer"] = plane_stats(got, same)
    if est is None:
        est = ON.estimate(cloud.positions, cloud.colors, weights.as_oracle_layers(),
                          weights.plan.levels)
    ref = OR.render_stream(est, view, ("rgb", "normal"))
    rec["e2e"] = plane_stats(got, ref)
    over = np.zeros(got["rgb"].shape[:2], dtype=bool)
    for p in PLANES:
        err = np.abs(got[p] - ref[p])
        over |= (err.max(axis=2) if err.ndim == 3 else err) > TOL
    if over.any():
        rec["e2e_over_pixels"] = explain_pixels(over, got, same, ref, gpu_sp, est, view)
    if levels:
        rec["levels"] = level_parity(dbg, est["vox"]["coords"])
    return rec


def replay_pixel(prep, x, y, alpha_max=OR.ALPHA_MAX, tile=16):
    """forward_kernel's blend sequence at one pixel (_raster_kernels.py:146-201)
    from a prepared frame: [(rank, point, alpha, T before)] of every splat that
    changes the pixel, in rank order, until T < 1/255."""
    tx, ty = x // tile, y // tile
    sx, sy, rad = prep["sx"], prep["sy"], prep["radius"]
    rect = tile_rects(sx, sy, rad, int(prep["ntx"]) * tile, int(prep["nty"]) * tile, tile)
    r1 = rad + 1.0
    with np.errstate(invalid="ignore", over="ignore"):
        hit = ((rect[:, 0] <= tx) & (tx <= rect[:, 1]) & (rect[:, 2] <= ty) & (ty <= rect[:, 3])
               & (np.ceil(sx - r1) <= x) & (x <= np.floor(sx + r1))
               & (np.ceil(sy - r1) <= y) & (y <= np.floor(sy + r1)))
        dx, dy = x - sx, y - sy
        hit &= ~(dx * dx + dy * dy > r1 * r1)
    ranks = np.nonzero(hit)[0]
    inv = prep["inv"]
    seq, t = [], 1.0
    for r in ranks.tolist():
        if t < OR.CUTOFF:
            break
        q = inv[r, 0] * dx[r] * dx[r] + 2.0 * inv[r, 1] * dx[r] * dy[r] + inv[r, 2] * dy[r] * dy[r]
        a = min(prep["opac"][r] * np.exp(-0.5 * q), alpha_max)
        if a < OR.CUTOFF:
            continue
        seq.append((r, int(prep["source"][r]), float(a), t))
        t *= 1.0 - a
    return seq


def classify(sg, so, p2v, depth_g, depth_o, alpha_of):
    """First divergence of two blend sequences at one pixel (GPU Gaussians vs
    oracle Gaussians, both through the oracle renderer). ``alpha_of(set,
    point)`` gives a point's alpha at the pixel under either parameter set.
    kinds: ``alpha_cutoff`` — a splat (with its whole run: a voxel's points
    share alpha) has alpha >= 1/255 under one set and < 1/255 under the other;
    ``T_cutoff`` — T crosses 1/255 one splat earlier under one set; ``order``
    — two splats blend in a different order; ``alpha`` — same splat, alphas
    differ by more than 1e-3."""
    c = OR.CUTOFF
    for k in range(max(len(sg), len(so))):
        if k >= len(sg) or k >= len(so):
            longer = "gpu" if len(sg) > len(so) else "oracle"
            short = so if longer == "gpu" else sg
            t_short = short[-1][3] * (1.0 - short[-1][2]) if short else 1.0
            t_long = (sg if longer == "gpu" else so)[k][3]
            return {"step": k, "kind": "T_cutoff", "longer": longer,
                    "T_gpu": t_long if longer == "gpu" else t_short,
                    "T_oracle": t_short if longer == "gpu" else t_long,
                    "straddle": bool(min(t_long, t_short) < c <= max(t_long, t_short)),
                    "rel_gap": abs(t_long - t_short) / c}
        (rg, pg, ag, tg), (ro, po, ao, to) = sg[k], so[k]
        if pg != po:
            in_o = {e[1] for e in so}
            in_g = {e[1] for e in sg}
            if pg not in in_o or po not in in_g:
                miss = pg if pg not in in_o else po
                a_g, a_o = alpha_of("gpu", miss), alpha_of("oracle", miss)
                return {"step": k, "kind": "alpha_cutoff", "point": miss, "voxel": int(p2v[miss]),
                        "alpha_gpu": a_g, "alpha_oracle": a_o,
                        "straddle": bool(min(a_g, a_o) < c <= max(a_g, a_o)),
                        "rel_gap": abs(a_g - a_o) / c}
            return {"step": k, "kind": "order", "gpu_point": pg, "oracle_point": po,
                    "gpu_voxel": int(p2v[pg]), "oracle_voxel": int(p2v[po]),
                    "depth_gpu": [float(depth_g[pg]), float(depth_g[po])],
                    "depth_oracle": [float(depth_o[pg]), float(depth_o[po])]}
        if abs(ag - ao) > 1e-3:
            return {"step": k, "kind": "alpha", "point": pg, "alpha": [ag, ao]}
    return {"kind": "none"}


def _alpha_at(prep, rank_of, point, x, y, alpha_max=OR.ALPHA_MAX):
    r = rank_of.get(point)
    if r is None:
        return 0.0
    dx, dy = x - prep["sx"][r], y - prep["sy"][r]
    inv = prep["inv"][r]
    q = inv[0] * dx * dx + 2.0 * inv[1] * dx * dy + inv[2] * dy * dy
    return float(min(prep["opac"][r] * np.exp(-0.5 * q), alpha_max))


def explain_pixels(over, got, same, ref, gpu_sp, est, view, limit=200) -> dict:
    """Attribute end-to-end pixels over 2e-3: renderer (GPU vs oracle on the
    GPU's own Gaussians) or parameters (oracle renderer on GPU vs oracle
    Gaussians), and for each pixel (up to ``limit``) the first divergence of
    the two blend sequences (``classify``)."""
    ys, xs = np.nonzero(over)
    ren = max(float(np.abs(got[p][ys, xs] - same[p][ys, xs]).max()) for p in PLANES)
    par = max(float(np.abs(same[p][ys, xs] - ref[p][ys, xs]).max()) for p in PLANES)
    pg, po = same["prep"], ref["prep"]
    p2v = est["vox"]["point_to_voxel"]
    dg = np.zeros(len(p2v))
    dg[pg["source"]] = pg["depth"]
    do = np.zeros(len(p2v))
    do[po["source"]] = po["depth"]
    rank_g = {int(p): r for r, p in enumerate(pg["source"])} if over.sum() else {}
    rank_o = {int(p): r for r, p in enumerate(po["source"])} if over.sum() else {}
    kinds, samples = {}, []
    for y, x in list(zip(ys.tolist(), xs.tolist()))[:limit]:
        def alpha_of(which, point):
            return _alpha_at(pg if which == "gpu" else po, rank_g if which == "gpu" else rank_o,
                             point, x, y)
        c = classify(replay_pixel(pg, x, y), replay_pixel(po, x, y), p2v, dg, do, alpha_of)
        c.update(y=y, x=x)
        kinds[c["kind"]] = kinds.get(c["kind"], 0) + 1
        samples.append(c)
    return {"count": int(over.sum()), "renderer_max_abs_there": ren,
            "parameter_effect_max_abs_there": par, "kinds": kinds,
            "all_threshold_crossings": all(c["kind"] in ("alpha_cutoff", "T_cutoff")
                                           and c["straddle"] and c["rel_gap"] < 5e-2
                                           for c in samples),
            "max_rel_gap": max((c.get("rel_gap", 0.0) for c in samples), default=0.0),
            "samples": samples}
