"""Time the REAL reference CPU path (splatforge, numpy + numba, imported
read-only from /root/reference — build container only, it does not travel to
the GPU box) next to this repo's oracle port on the same host and inputs.

BASELINE.md §3 protocol: P = estimators.estimate_neural, R = rasterizer.render
for rgb and for normal, one warm-up (numba JIT), then the median of `reps`;
NUMBA_NUM_THREADS / OPENBLAS_NUM_THREADS set explicitly (reported). Config 1
at 1 thread and at all threads; config 2 (one ring view) at all threads, R
timed once (≈ minutes per mode). Writes JSON (default
profiles/cpu_reference_r02.json).

usage: python tools/time_reference.py [out.json] [--skip-c2]
"""
import json
import os
import platform
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src")

CHILD = r'''
import json, sys, time, statistics
import numpy as np
sys.path.insert(0, ROOT)
from paper_2409_16504_b200 import scenes
from splatforge.pcio import PointCloud
from splatforge.estimators import EstimatorConfig, estimate_neural
from splatforge.sparsenet import NetworkPlan, init_random
from splatforge.gaussians import Camera
from splatforge.rasterizer import render
cfg_name, reps, r_reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cloud, views = scenes.config1() if cfg_name == "c1" else scenes.config2()
v = views[0]
cam = Camera(v.rotation, v.translation, v.fx, v.fy, v.cx, v.cy, v.width, v.height)
pc = PointCloud(cloud.positions, cloud.colors)
w = init_random(NetworkPlan(), 0)
cfg = EstimatorConfig(kind="neural")
sp = estimate_neural(pc, w, cfg)          # warm-up (numba JIT)
if r_reps > 1:
    render(sp, cam, "rgb"); render(sp, cam, "normal")
else:
    small = scenes.config1()[1][0]
    scam = Camera(small.rotation, small.translation, small.fx, small.fy, small.cx, small.cy,
                  small.width, small.height)
    s1 = scenes.config1()[0]
    ssp = estimate_neural(PointCloud(s1.positions, s1.colors), w, cfg)
    render(ssp, scam, "rgb"); render(ssp, scam, "normal")   # JIT on the small frame
P = []
for _ in range(reps):
    t = time.perf_counter(); sp = estimate_neural(pc, w, cfg); P.append(time.perf_counter() - t)
R = {"rgb": [], "normal": []}
for _ in range(r_reps):
    for m in R:
        t = time.perf_counter(); render(sp, cam, m); R[m].append(time.perf_counter() - t)
out = {"points": len(pc), "width": v.width, "height": v.height,
       "P_s": statistics.median(P), "P_samples": P,
       "R_rgb_s": statistics.median(R["rgb"]), "R_normal_s": statistics.median(R["normal"]),
       "R_samples": R}
out["frame_s"] = out["P_s"] + out["R_rgb_s"] + out["R_normal_s"]
print("RESULT " + json.dumps(out), flush=True)
'''

PORT = r'''
import json, sys, time, statistics
sys.path.insert(0, ROOT)
from oracle import net as ON, raster as OR
from paper_2409_16504_b200 import netplan, scenes
cfg_name, reps = sys.argv[1], int(sys.argv[2])
cloud, views = scenes.config1() if cfg_name == "c1" else scenes.config2()
w = netplan.init_random(netplan.NetworkPlan(), 0)
OR.build()
T = []
for _ in range(reps):
    t0 = time.perf_counter()
    est = ON.estimate(cloud.positions, cloud.colors, w.as_oracle_layers(), 3)
    t1 = time.perf_counter()
    for m in ("rgb", "normal"):
        OR.render_banded(est, views[0], m)
    T.append((t1 - t0, time.perf_counter() - t1))
print("RESULT " + json.dumps({"P_s": statistics.median(a for a, b in T),
                              "R_s": statistics.median(b for a, b in T),
                              "frame_s": statistics.median(a + b for a, b in T)}), flush=True)
'''


def child(code, args, threads, ref=True):
    env = dict(os.environ, NUMBA_NUM_THREADS=str(threads), OPENBLAS_NUM_THREADS=str(threads),
               OMP_NUM_THREADS=str(threads), PYTHONDONTWRITEBYTECODE="1",
               NUMBA_CACHE_DIR="/tmp/nb_cache_ref")
    if ref:
        env["PYTHONPATH"] = str(REF)
    src = code.replace("ROOT", repr(str(ROOT)))
    r = subprocess.run([sys.executable, "-c", src, *map(str, args)], env=env, capture_output=True,
                       text=True, cwd="/tmp")
    for line in r.stdout.splitlines():
        if line.startswith("RESULT "):
            return json.loads(line[7:])
    raise RuntimeError(r.stderr[-3000:])


def main():
    out = Path(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else \
        ROOT / "profiles" / "cpu_reference_r02.json"
    cores = os.cpu_count()
    cpu = platform.processor() or ""
    try:
        cpu = [ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if "model name" in ln][0]
    except Exception:
        pass
    rep = {"host": {"cpu": cpu, "logical_cores": cores},
           "protocol": "one warm-up, median of reps; NUMBA/OPENBLAS/OMP threads as listed",
           "runs": []}
    for cfg, threads, reps, r_reps in (("c1", 1, 3, 3), ("c1", cores, 3, 3)):
        r = child(CHILD, [cfg, reps, r_reps], threads)
        r.update(config=cfg, threads=threads, impl="reference (splatforge, numba)")
        rep["runs"].append(r)
        print(json.dumps(r), flush=True)
        p = child(PORT, [cfg, reps], threads, ref=False)
        p.update(config=cfg, threads=threads, impl="oracle port (numpy + C/OpenMP)")
        rep["runs"].append(p)
        print(json.dumps(p), flush=True)
    if "--skip-c2" not in sys.argv:
        r = child(CHILD, ["c2", 1, 1], cores)
        r.update(config="c2 view 0", threads=cores, impl="reference (splatforge, numba)")
        rep["runs"].append(r)
        print(json.dumps(r), flush=True)
        p = child(PORT, ["c2", 1], cores, ref=False)
        p.update(config="c2 view 0", threads=cores, impl="oracle port (numpy + C/OpenMP)")
        rep["runs"].append(p)
        print(json.dumps(p), flush=True)
    out.write_text(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main()
