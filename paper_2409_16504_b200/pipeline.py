"""The fused real-time path: point cloud -> P2ENet -> splat planes in one call.

``render_frame`` is ``render_planes(estimate_neural(cloud), cam)`` without
materialising per-point Gaussians: the renderer projects the M0 per-voxel
Gaussians once, sorts points by (voxel depth, index) and composites each
voxel's points as one run (colours per point). Output planes are identical
to the two-step path. This is what ``bench.py`` times.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .gaussians import Camera
from .netplan import NetworkWeights
from .pcio import EmptyCloudError, PlyBody, PointCloud
from .rasterizer import _PLANE_BIT, FrameBuffer, RenderOptions, _alloc_planes
from .sparsenet import ensure_loaded
from .voxelgrid import device_bbox, lattice_scale, stage_cloud

# Host clouds are uploaded on a dedicated stream (one per device) into
# persistent per-lane staging buffers (two per lane, alternating), with their
# own library context (own scratch arena) for the bbox. ``stage`` only
# ENQUEUES the copies, the bbox reduction and the 48-byte read-back of the
# bbox into pinned memory; ``prepare_cloud`` later waits for that read-back
# alone. Staging frame i+1 before rendering frame i therefore keeps the copy
# engine busy while the host waits for frame i's bbox (the one host round
# trip per frame, which gives the bit-exact lattice scale). Fixed staging
# addresses also keep the lane's CUDA-graph cache hot (graphs are keyed by
# pointers).
_UPLOAD_LANE = 1 << 16
_BBOX_LANE = 1 << 17
_upload_streams = {}
# The bbox reduction and its 48-byte read-back run on a stream of their own:
# on the upload stream the read-back (a device->host copy, queued on the same
# copy engine as earlier frames' plane read-backs) would hold back the next
# frame's host->device copies behind it in stream order.
_bbox_streams = {}
_staging = {}   # (device, lane) -> {"k": next, "bufs": [[pos, col, done_ev, ply_bytes, bbox_words], ...]}


class StagedCloud:
    """A host cloud whose upload is in flight (see ``stage``)."""

    def __init__(self, pos, col, n, slot, bbox_ev, done_ev, words):
        self.pos, self.col, self.n, self.slot = pos, col, n, slot
        self.bbox_ev, self.done_ev, self.words = bbox_ev, done_ev, words

    def __len__(self) -> int:
        return self.n


def _decode_words(words: np.ndarray) -> np.ndarray:
    """Order-preserving bbox words -> float64 (inverse of the device encoding)."""
    u = words.astype(np.uint64)
    neg = (u >> np.uint64(63)) == 0
    bits = np.where(neg, ~u, u & np.uint64(0x7FFFFFFFFFFFFFFF))
    return bits.view(np.float64).copy()


def stage(cloud, lane: int = 0) -> StagedCloud:
    """Enqueue the upload of a host cloud (PointCloud or PlyBody) for ``lane``:
    positions H2D (or the PLY bytes + device decode), bbox + its read-back,
    colours H2D — no host synchronisation."""
    dev = torch.cuda.current_device()
    up = _upload_streams.get(dev)
    if up is None:
        up = _upload_streams[dev] = torch.cuda.Stream(device=dev)
        _bbox_streams[dev] = torch.cuda.Stream(device=dev)
    bb = _bbox_streams[dev]
    st = _staging.setdefault((dev, lane), {"k": 0, "bufs": [[None] * 6, [None] * 6]})
    slot = st["bufs"][st["k"]]
    if slot[5]:   # staged but not yet rendered: its data would be overwritten
        raise RuntimeError(f"both staging buffers of lane {lane} hold unrendered clouds: render "
                           "a staged cloud of this lane (or stage on another lane) first")
    ply = isinstance(cloud, PlyBody)
    n = len(cloud) if ply else int(cloud.positions.shape[0])
    if n == 0:
        raise EmptyCloudError("empty cloud has no bbox")
    st["k"] ^= 1
    grow = slot[0] is None or slot[0].shape[0] < n
    grow_ply = ply and (slot[3] is None or slot[3].numel() < cloud.raw.numel())
    if (grow or grow_ply) and slot[2] is not None:
        # the last frame that read these buffers may still be running on its
        # stream: the caching allocator could hand the freed blocks to the
        # next allocation of another stream, so wait before dropping them
        slot[2].synchronize()
    if grow:
        slot[0] = torch.empty((n, 3), dtype=torch.float64, device=dev)
        slot[1] = torch.empty((n, 3), dtype=torch.float64, device=dev)
    if grow_ply:
        slot[3] = torch.empty(cloud.raw.numel(), dtype=torch.uint8, device=dev)
    if slot[4] is None:
        slot[4] = torch.empty(6, dtype=torch.int64).pin_memory()
    pos, col = slot[0][:n], slot[1][:n]
    cur = torch.cuda.current_stream(dev)
    up.wait_stream(cur)   # inputs the caller just wrote on its stream
    if slot[2] is not None:
        up.wait_event(slot[2])   # the frame that last read this staging buffer
    uctx = _lib.context(lane=_UPLOAD_LANE + lane)
    bctx = _lib.context(lane=_BBOX_LANE + lane)

    def host(a):
        if isinstance(a, torch.Tensor):
            return a
        return torch.from_numpy(np.ascontiguousarray(a))
    with torch.cuda.stream(up):
        if ply:   # the file's bytes cross PCIe; widened to float64 on the device
            body = slot[3][:cloud.raw.numel()]
            body.copy_(cloud.raw, non_blocking=cloud.raw.is_pinned())
            layout = (_lib.I32 * 9)(*cloud.offsets)
            uctx.call("sfb_ply_decode", _lib.ptr(body), n, cloud.stride, layout, _lib.ptr(pos),
                      _lib.ptr(col), _lib.P(0))
            pos_ev = up.record_event()
        else:
            hp = host(cloud.positions)
            pos.copy_(hp, non_blocking=hp.is_pinned())
            pos_ev = up.record_event()
            hc = host(cloud.colors)
            col.copy_(hc, non_blocking=hc.is_pinned())
        done_ev = up.record_event()
    bb.wait_event(pos_ev)
    with torch.cuda.stream(bb):
        bctx.call("sfb_bbox_async", _lib.ptr(pos), n, _lib.ptr(slot[4]))
        bbox_ev = bb.record_event()
    slot[5] = True   # pending until a frame consumes it (prepare_cloud)
    return StagedCloud(pos, col, n, slot, bbox_ev, done_ev, slot[4])


def prepare_cloud(cloud, lane: int = 0):
    """Device positions/colours, point count, lattice scale and bbox of a cloud
    (host clouds go through the upload stream; a ``StagedCloud`` from
    ``stage`` is used as is); ``slot`` is the staging buffer whose done-event
    the caller records after its frame (None for device clouds)."""
    if not isinstance(cloud, (PlyBody, StagedCloud)) and cloud.on_device:
        pos, col = stage_cloud(cloud)
        lo_hi = device_bbox(pos, lane)
        n = int(pos.shape[0])
        return pos, col, n, lattice_scale(n, lo_hi), lo_hi, None
    sc = cloud if isinstance(cloud, StagedCloud) else stage(cloud, lane)
    sc.slot[5] = False   # consumed: the caller records the frame's done event next
    sc.bbox_ev.synchronize()   # the 48-byte read-back only
    lo_hi = _decode_words(sc.words.numpy().view(np.uint64))
    torch.cuda.current_stream().wait_event(sc.done_ev)
    return sc.pos, sc.col, sc.n, lattice_scale(sc.n, lo_hi), lo_hi, sc.slot


def render_frame(cloud: PointCloud, weights: NetworkWeights, cam: Camera,
                 planes=("rgb", "normal"), background=(0.0, 0.0, 0.0),
                 options: RenderOptions = None, out=None, lane: int = 0) -> FrameBuffer:
    """Cloud -> P2ENet -> planes. ``lane`` selects an independent library
    context (own arena and CUDA graphs): issue frames from different lanes on
    different torch streams and they overlap on the GPU."""
    ctx = ensure_loaded(weights, lane)
    options = options or RenderOptions()
    pos, col, n, s, lo_hi, slot = prepare_cloud(cloud, lane)
    bg = np.ascontiguousarray(np.asarray(background, dtype=np.float64).reshape(3))
    rgb, nrm, dep, trans = out if out is not None else _alloc_planes(cam, planes, pos.device)
    mask = 0
    for p in planes:
        mask |= _PLANE_BIT[p]
    c, o = cam.struct(), options.struct()
    try:
        ctx.call("sfb_frame", _lib.ptr(pos), _lib.ptr(col), n, s, lo_hi.ctypes.data_as(_lib.P),
                 _lib.ctypes.byref(c), _lib.ctypes.byref(o), mask, bg.ctypes.data_as(_lib.P),
                 _lib.ptr(rgb), _lib.ptr(nrm), _lib.ptr(dep), _lib.ptr(trans))
    finally:
        if slot is not None:   # the staging buffer is free once this frame (or the
            # part of it that was enqueued before an error) is done
            slot[2] = torch.cuda.current_stream().record_event()
    if rgb is None:
        rgb = torch.zeros((int(cam.height), int(cam.width), 3), dtype=torch.float32,
                          device=pos.device)
    return FrameBuffer(int(cam.width), int(cam.height), rgb, trans, bg, nrm, dep)


def stats(lane: int = 0) -> dict:
    """Sizes of the last call (kept splats, runs, pyramid entries, voxels per level)."""
    return _lib.context(lane=lane).stats()


def render_frame_debug(cloud, weights: NetworkWeights, cam: Camera, planes=("rgb", "normal"),
                       background=(0.0, 0.0, 0.0), options: RenderOptions = None,
                       levels: int = 4, lane: int = 0):
    """``render_frame`` plus the fused path's internal order, for parity tests:
    ``source`` (rank -> point over the kept points, rasterizer.py:105), the runs
    of identical geometry (start rank, point count, tile rect x0 x1 y0 y1 of
    _raster_kernels.py:123-130) and, per UNet level, the level coordinates and
    27-tap kernel map in the level's own row order (sparsenet.py:201-207)."""
    ctx = ensure_loaded(weights, lane)
    n = len(cloud)
    dev = torch.device("cuda", torch.cuda.current_device())
    source = torch.empty(n, dtype=torch.int64, device=dev)
    rs = torch.empty(n, dtype=torch.int32, device=dev)
    rc = torch.empty(n, dtype=torch.int32, device=dev)
    rr = torch.empty((n, 4), dtype=torch.int32, device=dev)
    lc = torch.empty((levels, n, 3), dtype=torch.int32, device=dev)
    lm = torch.empty((levels, 27, n), dtype=torch.int32, device=dev)
    ctx.lib.sfb_set_frame_debug(ctx.handle, n, _lib.ptr(source), _lib.ptr(rs), _lib.ptr(rc),
                                _lib.ptr(rr), levels, _lib.ptr(lc), _lib.ptr(lm))
    try:
        fb = render_frame(cloud, weights, cam, planes, background, options, lane=lane)
        torch.cuda.synchronize()
    finally:
        ctx.lib.sfb_set_frame_debug(ctx.handle, 0, None, None, None, None, 0, None, None)
    st = ctx.stats()
    kept, runs = st["kept"], st["runs"]
    vox = st["voxels"]
    out = {"source": source[:kept], "run_start": rs[:runs], "run_count": rc[:runs],
           "run_rect": rr[:runs], "kept": kept, "runs": runs,
           "level_coords": [lc[l, :vox[l]] for l in range(levels) if vox[l] > 0],
           "level_maps": [lm[l, :, :vox[l]] for l in range(levels) if vox[l] > 0]}
    return fb, out
