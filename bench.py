#!/usr/bin/env python
"""Benchmark: ms/frame (P2ENet + splat) at ~800k points, 1024^2; frames/s at N GPUs.

Workload (BASELINE.json configs[1], "config 2"): a seeded union of 5
ellipsoids on a 1024^3 grid (~800k occupied voxels, scenes.config2), the
reference P2ENet with seeded random-init weights (init_random(NetworkPlan(),0)),
rendered to RGB + normal (+ transmittance) at 1024x1024 from 8 ring views.
One step = one frame = the full fused path on device: bbox/lattice scale ->
voxelize -> UNet -> head -> projection -> depth sort -> runs/binning ->
compositing. Frames are independent: under torchrun every rank renders its own
frames (views round-robin), no data-path collective ("scaling": "weak").

Lines printed (rank 0, one JSON line):
  value      whole-job frames/s with inputs resident in HBM (device-timed,
             CUDA events per step, L2 flushed between steps, max over ranks)
  e2e        the same through the public API with pinned HOST buffers:
             H2D of the cloud + D2H of the planes inside every timed step
  roofline   dominant stage: algorithmic bytes / its CUDA-event time vs the
             measured HBM copy bandwidth (MEASURED_PEAKS.json)
  cpu_baseline  the CPU oracle port (tests-only restatement of the reference)
             on a bounded sample of one frame, rank 0 at N=1
``--impl reference`` times only that CPU port (the reference package itself is
pure Python/numba and cannot ship to the GPU box).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

# Frames in flight run on 10 lanes x 3 streams (main, side, aux) each: with the
# default 8 hardware work queues, streams share queues and a frame's side-stream
# kernels queue behind other lanes' work. Must be set before CUDA initialises.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ms/frame (P2ENet+splat) at ~800k pts, 1024²; frames/sec at 1/2/4/8 B200"
UNIT = "frames/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=("c2", "c1", "c3", "c4", "c5"), default="c2",
                    help="c2: the headline workload (BASELINE configs[1]); c4: the 64-frame "
                         "sequence, frames block-sharded over ranks; c5: the 2048^3 scene, 32 "
                         "views round-robin over ranks (both also report gather-inclusive fps)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-profile", action="store_true", help="skip the CUPTI launch count")
    ap.add_argument("--view", type=int, default=-1,
                    help="render only this view (profiling runs; default: views round-robin)")
    ap.add_argument("--cpu-frames", type=int, default=1,
                    help="full config-2 frames of the CPU port timed for cpu_baseline")
    ap.add_argument("--lanes", type=int, default=10, help="frames in flight per GPU (streams)")
    ap.add_argument("--stage-ahead", type=int, default=2,
                    help="host clouds: uploads enqueued this many frames ahead (< e2e lanes)")
    ap.add_argument("--e2e-lanes", type=int, default=8,
                    help="frames in flight in the e2e (host-buffer) legs (PCIe-bound; 20-frame "
                         "runs: 4/6/8/12 lanes 0.876/0.871/0.873/0.870-0.908 ms, 12 with outliers); "
                         "0: --lanes")
    ap.add_argument("--net-mode", choices=("tc_tf32x3", "tc_bf16", "simt_f32", "simt_f64"),
                    default="tc_tf32x3",
                    help="P2ENet arithmetic (tc_tf32x3: fp32-accurate parity mode)")
    return ap.parse_args()


def workload(name):
    from paper_2409_16504_b200 import scenes
    if name == "c1":
        cloud, views = scenes.config1()
    elif name == "c3":
        cloud, views = scenes.config3()
    else:
        cloud, views = scenes.config2()
    return cloud, views


def traffic(kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the committed
    `ncu --set full` capture summary (profiles/traffic.json), else None."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        d = json.loads(p.read_text()).get(kernel)
        if d:
            return d["dram_bytes_per_launch"]
    return None


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------- CPU oracle leg
def cpu_frame(cloud, view, weights, threads):
    """One WHOLE frame of the CPU port of the reference path (tests-only
    restatement, oracle/): voxelize + UNet + head (estimators.py:214-231, numpy
    BLAS), then render rgb and normal (rasterizer.py:152-166: projection, sort,
    support radius, bin_tiles + forward_kernel over all tile rows, in bands of 8
    rows for bounded memory; C/OpenMP on `threads` threads). Nothing is
    extrapolated."""
    from oracle import net as ON
    from oracle import raster as OR
    t0 = time.perf_counter()
    est = ON.estimate(cloud.positions, cloud.colors, weights.as_oracle_layers(),
                      weights.plan.levels)
    t1 = time.perf_counter()
    for mode in ("rgb", "normal"):
        OR.render_banded(est, view, mode)
    t2 = time.perf_counter()
    return dict(seconds=t2 - t0, p2enet_s=t1 - t0, render_s=t2 - t1)


def cpu_env():
    """Thread settings of the CPU legs (set before numpy / the oracle load)."""
    cores = os.cpu_count()
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        os.environ.setdefault(k, str(cores))
    cpu = ""
    try:
        cpu = [ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if "model name" in ln][0]
    except (OSError, IndexError):
        pass
    return cores, cpu


def workload_config(name, cloud, views):
    """The `config` keys both arms report for the same workload."""
    n = int(len(cloud.positions))
    W, H = int(views[0].width), int(views[0].height)
    scene = {"c1": "scenes.config1", "c3": "cube + torus, noisy, scenes.config3"}.get(
        name, "5-ellipsoid union, scenes.config2")
    return {"workload": f"{name}: {n} pts ({scene}), P2ENet "
                        f"init_random(seed 0) -> {W}x{H} rgb+normal+T, {len(views)} ring views",
            "points": n, "width": W, "height": H}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores, cpu = cpu_env()
    from oracle import raster as OR
    from paper_2409_16504_b200 import netplan, scenes
    OR.build()
    name = args.config if args.config in ("c1", "c2", "c3") else "c2"
    cloud, views = workload(name)
    w = netplan.init_random(netplan.NetworkPlan(), 0)
    # warm-up on a small frame (numpy / OpenMP / page-in), then whole frames of
    # the workload until K are done or the time budget (SFB_REF_BUDGET_S,
    # default 300 s) is spent — at least one
    if args.warmup:
        c1, v1 = scenes.config1(n_dirs=4000)
        cpu_frame(c1, v1[0], w, cores)
    budget = float(os.environ.get("SFB_REF_BUDGET_S", "300"))
    recs = []
    t_start = time.perf_counter()
    for i in range(args.steps):
        recs.append(cpu_frame(cloud, views[i % len(views)], w, cores))
        if time.perf_counter() - t_start > budget:
            break
    tot = sum(r["seconds"] for r in recs)
    value = len(recs) / tot
    sample = (f"oracle port (numpy + C/OpenMP restatement of the reference path), {len(recs)} "
              f"whole {name} frame(s): P2ENet {np.mean([r['p2enet_s'] for r in recs]):.2f} s + "
              f"render rgb+normal over all tile rows {np.mean([r['render_s'] for r in recs]):.2f} s "
              f"per frame; {cores} threads on {cpu or 'unknown CPU'}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(recs), "steps_sampled": len(recs),
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(name, cloud, views),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample, "cpu": cpu,
                         "p2enet_s": float(np.mean([r["p2enet_s"] for r in recs])),
                         "render_s": float(np.mean([r["render_s"] for r in recs]))},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- GPU leg
class ClockSampler:
    def __init__(self, gpu):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        self.skip = 0

    def mark(self):
        """Samples before this call (nvidia-smi start-up, idle clocks) are dropped."""
        self.f.flush()
        self.skip = len(Path(self.f.name).read_text().splitlines())

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        rows = [r.split(",") for r in Path(self.f.name).read_text().splitlines()[self.skip:]
                if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2409_16504_b200 import _lib, netplan
    from paper_2409_16504_b200.gaussians import Camera
    from paper_2409_16504_b200.pcio import PointCloud
    from paper_2409_16504_b200.pipeline import render_frame, stage, stats
    from paper_2409_16504_b200.pcio import PlyBody
    from paper_2409_16504_b200.service import CameraPose, render_pose_frame

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    from paper_2409_16504_b200.shard import max_over_ranks, unit_of

    cloud, views = workload(args.config)
    cams = [Camera.of(v) for v in views]
    poses = [CameraPose(c, "relit") for c in cams]   # render_pose requests (headlight)
    weights = netplan.init_random(netplan.NetworkPlan(), 0)
    from paper_2409_16504_b200 import sparsenet
    sparsenet.set_mode(args.net_mode)
    W, H = cams[0].width, cams[0].height
    planes = ("rgb", "normal")
    lanes = max(1, args.lanes)
    # inputs larger than L2: `copies` distinct device copies of the cloud (38 MB
    # each) are rotated, so consecutive frames never re-read a cached input
    # (one CUDA graph per (lane, copy): at most 32 copies, the graph cache size)
    copies = min(32, max(lanes + 1, 4, -(-140 * 10**6 // (48 * len(cloud)))))
    dev_clouds = [PointCloud(torch.from_numpy(cloud.positions).cuda(),
                             torch.from_numpy(cloud.colors).cuda(), validate=False)
                  for _ in range(copies)]
    streams = [torch.cuda.Stream() for _ in range(lanes)]

    def planes_buf():
        return (torch.empty((H, W, 3), dtype=torch.float32, device="cuda"),
                torch.empty((H, W, 3), dtype=torch.float32, device="cuda"), None,
                torch.empty((H, W), dtype=torch.float32, device="cuda"))
    # one output set per (lane, input copy) so the graph of a lane is keyed once per copy
    outs = [[planes_buf() for _ in range(copies)] for _ in range(lanes)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # 256 MB > 126 MB L2

    def view_of(i):   # views round-robin over ranks
        return cams[args.view if args.view >= 0 else unit_of(i, rank, world, len(cams))]

    rgba_out = None   # render_pose leg: one RGBA8 device frame per (lane, input copy)
    # device->host read-backs of the e2e legs: one stream per lane, so a frame's
    # read-back starts when that frame is done, not behind slower earlier ones
    downs = [torch.cuda.Stream() for _ in range(lanes)]
    down_done = {}

    active = [lanes]   # lanes the next batch uses (the e2e legs may use fewer)

    def issue(i, cloud_list, host_out=None, src=None):
        lane = i % active[0]
        k = i % copies
        src = cloud_list[k] if src is None else src
        with torch.cuda.stream(streams[lane]):
            if rgba_out is not None:   # service.render_pose streaming path (relit, RGBA8)
                fr = render_pose_frame(src, weights, poses[unit_of(i, rank, world, len(cams))],
                                       out=rgba_out[lane][k], lane=lane)
                host_out[lane][0].copy_(fr, non_blocking=True)
                return fr
            if (lane, k) in down_done:   # the previous read-back of these planes
                streams[lane].wait_event(down_done.pop((lane, k)))
            fb = render_frame(src, weights, view_of(i), planes, out=outs[lane][k], lane=lane)
            if host_out is not None:   # read-back on the lane's download stream
                down = downs[lane]
                down.wait_stream(streams[lane])
                with torch.cuda.stream(down):
                    ho = host_out[lane]
                    ho[0].copy_(fb.rgb, non_blocking=True)
                    ho[1].copy_(fb.normal, non_blocking=True)
                    ho[2].copy_(fb.transmittance, non_blocking=True)
                    down_done[(lane, k)] = down.record_event()
        return fb

    def run_batch(n_frames, cloud_list, host_out=None):
        """n_frames frames over the lanes; device time between a start event on
        the default stream and the join of every lane."""
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        start.record(cur)
        for st in streams:
            st.wait_stream(cur)
        h0 = time.perf_counter()
        host_in = not (isinstance(cloud_list[0], PointCloud) and cloud_list[0].on_device)
        # host inputs: the uploads of frames i+1 and i+2 are enqueued
        # (pipeline.stage) before frame i waits for its bbox, so the copy
        # engine has ~2 frames of work queued and host hiccups do not idle it
        # (frames i and i+ahead must not share a lane: a lane has two staging buffers)
        nl = active[0]
        ahead = min(args.stage_ahead, nl - 1) if nl >= 3 else 1
        staged = [stage(cloud_list[j % copies], j % nl) for j in range(min(ahead, n_frames))] \
            if host_in else []
        for i in range(n_frames):
            cur_src = staged.pop(0) if host_in else None
            if host_in and i + ahead < n_frames:
                staged.append(stage(cloud_list[(i + ahead) % copies], (i + ahead) % nl))
            issue(i, cloud_list, host_out, cur_src)
        host = time.perf_counter() - h0
        for st in streams + downs:
            cur.wait_stream(st)
        end.record(cur)
        end.synchronize()
        return start.elapsed_time(end), host

    # warm-up: every (lane, copy) pair runs eager -> capture -> replay
    for _ in range(max(args.warmup, 3)):
        run_batch(lanes * copies, dev_clouds)
    barrier()

    # ---- latency: one frame at a time, L2 flushed between frames (lane 0)
    n_lat = min(args.steps, 50)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(n_lat)]
    for i in range(n_lat):
        flush.zero_()
        with torch.cuda.stream(streams[0]):
            streams[0].wait_stream(torch.cuda.current_stream())
        evs[i][0].record(streams[0])
        with torch.cuda.stream(streams[0]):   # lane 0's input copies (graphs captured in warm-up)
            k = (i * lanes) % copies
            render_frame(dev_clouds[k], weights, view_of(i), planes, out=outs[0][k], lane=0)
        evs[i][1].record(streams[0])
        torch.cuda.current_stream().wait_stream(streams[0])
    torch.cuda.synchronize()
    lat_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in evs) / n_lat)

    # ---- timed region: throughput, frames overlapped over the lanes. The
    # clock sampler (50 ms period) watches a >= 1 s window of this same load
    # around it: the timed K frames take only milliseconds
    barrier()
    clocks = ClockSampler(local)
    time.sleep(0.5)   # nvidia-smi needs a moment before its first sample
    clocks.mark()
    t_mark = time.perf_counter()
    while time.perf_counter() - t_mark < 0.5:   # load before the timed region
        run_batch(lanes * copies, dev_clouds)
    barrier()
    ms, host_s = run_batch(args.steps, dev_clouds)
    barrier()
    while time.perf_counter() - t_mark < 1.0:   # and after it
        run_batch(lanes * copies, dev_clouds)
    clk = clocks.stop()
    ms_max = max_over_ranks(ms)
    value = world * args.steps / (ms_max / 1e3)
    st = stats()

    # ---- per-stage CUDA-event times (eager launches, outside the timed region)
    ctx = _lib.context()
    ctx.set_timing(True)
    stage_acc = {}
    comp_by_view = {}
    n_stage = min(args.steps, 16)
    for i in range(n_stage):
        flush.zero_()
        render_frame(dev_clouds[0], weights, view_of(i), planes, out=outs[0][0])
        for k, v in ctx.stage_times().items():
            stage_acc[k] = stage_acc.get(k, 0.0) + v
            if k == "composite_reps":   # the compositor's cost depends on the view
                vid = args.view if args.view >= 0 else unit_of(i, rank, world, len(cams))
                comp_by_view.setdefault(vid, []).append(v / _lib.COMPOSITE_REPS)
    ctx.set_timing(False)
    stage_ms = {k: v / n_stage for k, v in stage_acc.items()}
    stage_ms.pop("untimed", None)
    if "composite_reps" in stage_ms:   # per-launch duration of the compositor kernel
        stage_ms["composite_kernel"] = stage_ms.pop("composite_reps") / _lib.COMPOSITE_REPS
    comp_by_view = {u: sum(v) / len(v) for u, v in sorted(comp_by_view.items())}

    # ---- e2e: public API with pinned HOST buffers, copies inside every step
    e2e = None
    if not args.no_e2e:
        # PCIe-bound legs: fewer frames in flight than the device leg keeps the
        # copy engines' queues short (a short run ends sooner after its last upload)
        active[0] = max(1, min(lanes, args.e2e_lanes or lanes))
        host_clouds = [PointCloud(torch.from_numpy(cloud.positions).pin_memory(),
                                  torch.from_numpy(cloud.colors).pin_memory(), validate=False)
                       for _ in range(copies)]
        host_out = [[torch.empty((H, W, 3), dtype=torch.float32).pin_memory(),
                     torch.empty((H, W, 3), dtype=torch.float32).pin_memory(),
                     torch.empty((H, W), dtype=torch.float32).pin_memory()] for _ in range(lanes)]
        h2d = host_clouds[0].positions.nbytes + host_clouds[0].colors.nbytes
        d2h = sum(x.nbytes for x in host_out[0])
        for _ in range(6):   # every (lane, input copy, staging buffer) graph captured
            run_batch(lanes * copies, host_clouds, host_out)
        barrier()
        ms2, _ = run_batch(args.steps, host_clouds, host_out)
        barrier()
        ms2 = max_over_ranks(ms2)
        e2e = {"value": world * args.steps / (ms2 / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": ms2 / args.steps, "lanes": active[0]}
        # the streaming caller (service.render_pose, mode relit): same host
        # clouds in, one RGBA8 frame out per step (4 bytes/px instead of 28)
        rgba_out = [[torch.empty((H, W, 4), dtype=torch.uint8, device="cuda")
                     for _ in range(copies)] for _ in range(lanes)]
        host_rgba = [[torch.empty((H, W, 4), dtype=torch.uint8).pin_memory()] for _ in range(lanes)]
        for _ in range(6):
            run_batch(lanes * copies, host_clouds, host_rgba)
        barrier()
        ms3, _ = run_batch(args.steps, host_clouds, host_rgba)
        barrier()
        ms3 = max_over_ranks(ms3)
        e2e["render_pose_relit_rgba8"] = {
            "value": world * args.steps / (ms3 / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(host_rgba[0][0].nbytes), "ms_per_step": ms3 / args.steps}
        # the same streaming call fed the binary PLY body a client would send
        # (15 B/point; config-2 positions are integer voxels and colours
        # uint8/255, so the decoded cloud is bit-identical to the float64 one)
        ply_clouds = [PlyBody.from_cloud(cloud) for _ in range(copies)]
        for _ in range(6):
            run_batch(lanes * copies, ply_clouds, host_rgba)
        barrier()
        ms4, _ = run_batch(args.steps, ply_clouds, host_rgba)
        barrier()
        ms4 = max_over_ranks(ms4)
        e2e["render_pose_relit_rgba8_from_ply"] = {
            "value": world * args.steps / (ms4 / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": int(ply_clouds[0].raw.numel()),
            "d2h_bytes_per_step": int(host_rgba[0][0].nbytes), "ms_per_step": ms4 / args.steps}
        rgba_out = None
        active[0] = lanes

    # ---- kernel launches of one frame (CUPTI via torch.profiler, outside the timed region)
    launches = None
    if args.no_profile:
        launches = "not counted (--no-profile)"
    else:
        try:
            from torch.profiler import ProfilerActivity, profile
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                render_frame(dev_clouds[0], weights, view_of(0), planes, out=outs[0][0])
                torch.cuda.synchronize()
            launches = sum(1 for e in prof.events() if e.device_type.name == "CUDA"
                           and "memcpy" not in e.name.lower() and "memset" not in e.name.lower())
        except Exception as exc:  # pragma: no cover
            launches = f"unavailable: {exc}"

    # ---- roofline of the dominant stage
    hbm, hbm_kind = peaks()
    n = len(cloud)
    px = W * H
    m0 = st["voxels"][0]
    # the unit is one frame; algorithmic bytes per frame
    # B_frame = 48*N (read the fp64 cloud) + 28*W*H (write rgb + normal + T,
    # f32); the fused path never writes per-point Gaussians, so §8(d)'s 68*N
    # term is dropped. One k_composite launch processes one frame.
    b_frame = 48 * n + 28 * px
    kb = {   # bytes each stage must move, for the per-stage GB/s
        "voxelize": 48 * n + 16 * n + (9 * 8 + 12) * m0,
        "sort": st["kept"] * (4 + 4) * 2,
        "composite": 28 * px + 128 * st["runs"],
        "project": 14 * 8 * m0 + 8 * 8 * m0,
    }
    # The dominant single kernel of the frame is k_composite (the composite
    # stage is exactly that one launch; profiles/ holds the launch list). The
    # UNet stage is a chain of ~40 small launches, not one kernel.
    # its per-launch duration: four back-to-back launches between CUDA events on
    # the lane stream in stage-timing mode (the eager frame's own "composite"
    # interval also holds host launch gaps); profiles/README.md compares it with
    # the ncu launch list
    kern = "composite_kernel" if "composite_kernel" in stage_ms else "composite"
    kb["composite_kernel"] = kb["composite"]
    roof = None
    if kern in stage_ms:
        ach = b_frame / (stage_ms[kern] / 1e3) / 1e9
        roof = {"kernel": "k_composite", "bound": "hbm", "achieved": ach, "peak": hbm,
                "unit": "GB/s", "frac": ach / hbm, "traffic": traffic("k_composite"),
                "peak_kind": hbm_kind, "algorithmic_bytes": b_frame,
                "algorithmic_bytes_formula": "48*N + 28*W*H per frame (SURVEY.md 8(d), fused path)",
                "ms": stage_ms[kern],
                "frame": {"ms": ms_max / args.steps,
                          "GB/s": b_frame / (ms_max / args.steps / 1e3) / 1e9},
                "stages": {k: {"ms": stage_ms[k], "bytes": kb[k],
                               "GB/s": kb[k] / (stage_ms[k] / 1e3) / 1e9}
                           for k in kb if k in stage_ms}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores, cpu_name = cpu_env()
        recs = [cpu_frame(cloud, views[i % len(views)], weights, cores)
                for i in range(max(1, args.cpu_frames))]
        tot = sum(r["seconds"] for r in recs)
        cpu = {"value": len(recs) / tot, "unit": UNIT, "cores": cores, "kind": "port",
               "cpu": cpu_name,
               "sample": (f"oracle port, {len(recs)} whole frame(s) of this workload: P2ENet "
                          f"{np.mean([r['p2enet_s'] for r in recs]):.2f} s + render rgb+normal "
                          f"(all tile rows) {np.mean([r['render_s'] for r in recs]):.2f} s; "
                          f"{tot / len(recs):.1f} s/frame on {cores} threads")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {**workload_config(args.config, cloud, cams), "voxels": m0,
                       "parallelism": f"frames x{world} (no collective)",
                       "lanes_per_gpu": lanes,
                       "l2": (f"timed region: {copies} distinct {48 * n / 1e6:.0f} MB input copies "
                              f"rotated ({copies * 48 * n / 1e6:.0f} MB; L2 126 MB), frames "
                              f"overlapped on {lanes} streams; latency: 256 MB L2 flush between "
                              "frames"),
                       "net_arithmetic": {"tc_tf32x3": "tcgen05 tf32 hi/lo split (fp32-accurate)",
                                          "tc_bf16": "tcgen05 bf16 operands, fp32 accumulation",
                                          "simt_f32": "fp32 FFMA",
                                          "simt_f64": "fp64 SIMT (reference arithmetic)"}[args.net_mode]
                                         + " convs; fp64 geometry / compositing"},
            "latency_ms_per_frame": lat_ms,
            "e2e": e2e, "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu,
            "clocks": clk, "stages_ms_eager": stage_ms, "composite_ms_by_view": comp_by_view,
            "stats": st,
            "host_enqueue_ms_per_step": 1e3 * host_s / args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------- sharded jobs (c4 / c5)
def sharded_job(n_units, policy, render_unit, rank, world, lanes=1):
    """This rank's shard of a job of independent units:
    ``render_unit(u, lane)`` renders unit u and returns its planes; units go
    round the lanes (streams). No data-path collective; the planes are
    gathered afterwards (shard.gather_planes)."""
    from paper_2409_16504_b200.shard import shard
    return {u: render_unit(u, i % lanes)
            for i, u in enumerate(shard(n_units, rank, world, policy))}


def run_units(args):
    """c4 (64-frame sequence, frames block-sharded) / c5 (2048^3 scene, 32
    views round-robin): every rank renders its own units end to end (P2ENet +
    splat per unit). ``value`` = units/s from device time (max over ranks);
    ``gather`` = units/s of the wall-clock job including each rank's
    device->host copies of its planes (``local``) and the planes of every
    unit delivered to rank 0's host memory (``to_rank0``: NCCL point-to-point
    over NVLink, then rank 0's copies), max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2409_16504_b200 import netplan, scenes
    from paper_2409_16504_b200.gaussians import Camera
    from paper_2409_16504_b200.pcio import PointCloud
    from paper_2409_16504_b200.pipeline import render_frame, stats
    from paper_2409_16504_b200.shard import gather_planes, max_over_ranks, shard

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    weights = netplan.init_random(netplan.NetworkPlan(), 0)
    from paper_2409_16504_b200 import sparsenet
    sparsenet.set_mode(args.net_mode)
    if args.config == "c4":
        n_units, policy = 64, "block"
        mine = shard(n_units, rank, world, policy)
        clouds, cams = {}, {}
        for u in mine:
            c, v = scenes.config4_frame(u)
            clouds[u] = PointCloud(torch.from_numpy(c.positions).cuda(),
                                   torch.from_numpy(c.colors).cuda(), validate=False)
            cams[u] = Camera.of(v[0])
        points = int(np.mean([len(clouds[u]) for u in mine]))
        desc = (f"c4: 64-frame sequence of the 5-ellipsoid union (scenes.config4_frame, ~{points} "
                f"pts/frame), one 1024x1024 view per frame, frames block-sharded over ranks")
    else:
        c, views = scenes.config5()
        n_units, policy = len(views), "round_robin"
        mine = shard(n_units, rank, world, policy)
        dev = PointCloud(torch.from_numpy(c.positions).cuda(), torch.from_numpy(c.colors).cuda(),
                         validate=False)
        clouds = {u: dev for u in mine}
        cams = {u: Camera.of(views[u]) for u in mine}
        points = len(c)
        desc = (f"c5: 2048^3 terrain + 50 boxes ({points} pts, scenes.config5), 32 views at "
                f"1920x1080 round-robin over ranks, P2ENet + splat per view")
    # c5 frames are ~7x larger (5.6 M points; each lane's scratch arena is ~3 GB):
    # measured 1.23 / 0.97 / 0.93 ms per view on 2 / 4 / 8 lanes; SFB_C5_LANES overrides
    c5_lanes = int(os.environ.get("SFB_C5_LANES", "8"))
    lanes = max(1, min(args.lanes if args.config == "c4" else min(args.lanes, c5_lanes), len(mine) or 1))
    streams = [torch.cuda.Stream() for _ in range(lanes)]
    downs = [torch.cuda.Stream() for _ in range(lanes)]
    outs = {}
    for u in mine:
        H, W = cams[u].height, cams[u].width
        outs[u] = (torch.empty((H, W, 3), dtype=torch.float32, device="cuda"),
                   torch.empty((H, W, 3), dtype=torch.float32, device="cuda"),
                   None, torch.empty((H, W), dtype=torch.float32, device="cuda"))
    host = {u: tuple(torch.empty(t.shape, dtype=t.dtype).pin_memory()
                     for t in (outs[u][0], outs[u][1], outs[u][3])) for u in mine}
    # rank 0's pinned destination of every unit's planes for the gather
    shape_of = {u: (cams[u].height, cams[u].width) for u in mine}
    ref_hw = next(iter(shape_of.values()))
    gather_out = ({u: (torch.empty(ref_hw + (3,), dtype=torch.float32).pin_memory(),
                       torch.empty(ref_hw + (3,), dtype=torch.float32).pin_memory(),
                       torch.empty(ref_hw, dtype=torch.float32).pin_memory())
                   for u in range(n_units)} if rank == 0 else None)

    def render_unit(u, lane):
        with torch.cuda.stream(streams[lane]):
            fb = render_frame(clouds[u], weights, cams[u], ("rgb", "normal"), out=outs[u],
                              lane=lane)
        return (fb.rgb, fb.normal, fb.transmittance)

    def job(copy_back=False):
        cur = torch.cuda.current_stream()
        for st in streams:
            st.wait_stream(cur)
        planes = sharded_job(n_units, policy, render_unit, rank, world, lanes)
        if copy_back:   # each rank's planes into pinned host memory, per lane
            for i, u in enumerate(mine):
                lane = i % lanes
                downs[lane].wait_stream(streams[lane])
                with torch.cuda.stream(downs[lane]):
                    for h, t in zip(host[u], planes[u]):
                        h.copy_(t, non_blocking=True)
        for st in streams + downs:
            cur.wait_stream(st)
        return planes

    for _ in range(max(args.warmup, 3)):   # eager -> capture -> replay per (lane, unit)
        job(copy_back=True)
    barrier()
    clocks = ClockSampler(local)
    time.sleep(0.5)
    clocks.mark()
    t_mark = time.perf_counter()
    while time.perf_counter() - t_mark < 0.5:
        job()
    barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    reps = max(1, args.steps // max(1, n_units))
    for _ in range(reps):
        job()
    end.record()
    end.synchronize()
    ms = max_over_ranks(start.elapsed_time(end))
    barrier()
    while time.perf_counter() - t_mark < 1.0:
        job()
    clk = clocks.stop()
    # gather-inclusive wall clock (host timer around the whole job, max over ranks)
    barrier()
    t0 = time.perf_counter()
    planes = job(copy_back=True)
    torch.cuda.synchronize()
    t_local = max_over_ranks(time.perf_counter() - t0)
    barrier()
    t0 = time.perf_counter()
    planes = job()
    merged = gather_planes(planes, dst=0, host=True, out=gather_out)
    t_rank0 = max_over_ranks(time.perf_counter() - t0)
    st = stats()
    if rank == 0:
        assert sorted(merged) == list(range(n_units)), "gather lost or duplicated units"
        per_unit = sum(t.nbytes for t in merged[0])
        total_units = n_units * reps
        print(json.dumps({
            "metric": METRIC, "value": total_units / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": total_units, "warmup": args.warmup, "ms_per_step": ms / total_units,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": desc, "points": points, "units": n_units, "policy": policy,
                       "parallelism": f"units x{world} (no collective on the data path)",
                       "lanes_per_gpu": lanes, "passes_timed": reps},
            "gather": {"local_units_per_s": n_units / t_local,
                       "to_rank0_units_per_s": n_units / t_rank0,
                       "bytes_per_unit": per_unit,
                       "note": "wall clock of one pass including the device->host copies of "
                               "every unit's rgb+normal+T f32 planes (local: each rank into its "
                               "own pinned memory; to_rank0: all planes in rank 0's host "
                               "memory via NCCL p2p + copies)"},
            "clocks": clk, "stats": st,
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.config in ("c4", "c5"):
        run_units(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
