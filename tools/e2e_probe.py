"""Where the e2e leg loses against the PCIe bound: ms/frame of
  copies  : the frame's copies alone (H2D cloud on one stream, D2H planes on another)
  up      : host clouds in, planes stay on the device
  down    : device clouds in, planes read back
  full    : host clouds in, planes read back (bench.py's e2e leg)
with 8 lanes, one-frame-ahead staging as in bench.py."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2409_16504_b200 import netplan, scenes
from paper_2409_16504_b200.gaussians import Camera
from paper_2409_16504_b200.pcio import PointCloud
from paper_2409_16504_b200.pipeline import render_frame, stage

lanes, copies = 8, 9
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
cloud, views = scenes.config2()
w = netplan.init_random(netplan.NetworkPlan(), 0)
cams = [Camera.of(v) for v in views]
H = W = 1024
host = [PointCloud(torch.from_numpy(cloud.positions).pin_memory(), torch.from_numpy(cloud.colors).pin_memory(),
                   validate=False) for _ in range(copies)]
dev = [PointCloud(torch.from_numpy(cloud.positions).cuda(), torch.from_numpy(cloud.colors).cuda(), validate=False)
       for _ in range(copies)]
streams = [torch.cuda.Stream() for _ in range(lanes)]
down = torch.cuda.Stream()
outs = [[(torch.empty((H, W, 3), device="cuda"), torch.empty((H, W, 3), device="cuda"), None,
          torch.empty((H, W), device="cuda")) for _ in range(copies)] for _ in range(lanes)]
hout = [[torch.empty((H, W, 3)).pin_memory(), torch.empty((H, W, 3)).pin_memory(),
         torch.empty((H, W)).pin_memory()] for _ in range(lanes)]


done = {}


def run(n, src, readback, bench_waits=False):
    cur = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cur)
    for s in streams:
        s.wait_stream(cur)
    hostin = not src[0].on_device
    nxt = stage(src[0], 0) if hostin else None
    for i in range(n):
        lane, k = i % lanes, i % copies
        cs = nxt
        if hostin and i + 1 < n:
            nxt = stage(src[(i + 1) % copies], (i + 1) % lanes)
        with torch.cuda.stream(streams[lane]):
            if bench_waits and (lane, k) in done:
                streams[lane].wait_event(done.pop((lane, k)))
            fb = render_frame(cs if hostin else src[k], w, cams[i % len(cams)], out=outs[lane][k], lane=lane)
            if readback:
                down.wait_stream(streams[lane])
                with torch.cuda.stream(down):
                    hout[lane][0].copy_(fb.rgb, non_blocking=True)
                    hout[lane][1].copy_(fb.normal, non_blocking=True)
                    hout[lane][2].copy_(fb.transmittance, non_blocking=True)
                    if bench_waits:
                        done[(lane, k)] = down.record_event()
                if not bench_waits:
                    streams[lane].wait_stream(down)
    for s in streams + [down]:
        cur.wait_stream(s)
    b.record(cur)
    b.synchronize()
    return a.elapsed_time(b) / n


def copies_only(n):
    up = torch.cuda.Stream()
    dpos = [torch.empty_like(host[0].positions, device="cuda") for _ in range(2)]
    dcol = [torch.empty_like(host[0].colors, device="cuda") for _ in range(2)]
    cur = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cur)
    up.wait_stream(cur); down.wait_stream(cur)
    for i in range(n):
        with torch.cuda.stream(up):
            dpos[i & 1].copy_(host[i % copies].positions, non_blocking=True)
            dcol[i & 1].copy_(host[i % copies].colors, non_blocking=True)
        with torch.cuda.stream(down):
            o = outs[i % lanes][0]
            hout[i % lanes][0].copy_(o[0], non_blocking=True)
            hout[i % lanes][1].copy_(o[1], non_blocking=True)
            hout[i % lanes][2].copy_(o[3], non_blocking=True)
    cur.wait_stream(up); cur.wait_stream(down)
    b.record(cur)
    b.synchronize()
    return a.elapsed_time(b) / n


for _ in range(4):
    run(lanes * copies, host, True)
    run(lanes * copies, dev, True)
copies_only(20)
res = {}
for r in range(2):
    res.setdefault("copies", []).append(copies_only(steps))
    res.setdefault("device", []).append(run(steps, dev, False))
    res.setdefault("up", []).append(run(steps, host, False))
    res.setdefault("down", []).append(run(steps, dev, True))
    res.setdefault("full", []).append(run(steps, host, True))
    res.setdefault("full_bench_waits", []).append(run(steps, host, True, True))
    res.setdefault("down_bench_waits", []).append(run(steps, dev, True, True))
for k, v in res.items():
    print(f"{k:8s} " + " ".join(f"{x:.4f}" for x in v) + " ms/frame")
