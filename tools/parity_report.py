"""Full-frame parity report of the fused GPU frame vs the CPU oracle, every
BASELINE config (tests/parity_util.py): order / rect / offset exactness,
UNet level maps, and per-plane max |d| and pixels over 2e-3 on identical
Gaussians and end to end. Writes JSON (default gpurun_out/parity.json).

usage: python tools/parity_report.py [out.json] [--c4-frames N] [--c5-views N]
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import net as ON  # noqa: E402
from paper_2409_16504_b200 import netplan, scenes  # noqa: E402
from paper_2409_16504_b200.pcio import PointCloud  # noqa: E402
from parity_util import frame_parity, gpu_splats_np  # noqa: E402


def run(cloud, views, w, which, name, levels_for=(0,)):
    pc = PointCloud(cloud.positions, cloud.colors)
    est = ON.estimate(cloud.positions, cloud.colors, w.as_oracle_layers(), 3)
    sp = gpu_splats_np(pc, w)
    out = []
    for k in which:
        t = time.time()
        rec = frame_parity(pc, cloud, w, views[k], est=est, gpu_sp=sp, levels=k in levels_for)
        rec.update(view=int(k), points=len(cloud), seconds=round(time.time() - t, 2))
        out.append(rec)
        print(name, k, json.dumps({x: rec[x] for x in ("order", "renderer", "e2e")}), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out", nargs="?", default=str(ROOT / "gpurun_out" / "parity.json"))
    ap.add_argument("--c4-frames", type=int, default=64)
    ap.add_argument("--c5-views", type=int, default=32)
    ap.add_argument("--c3-views", type=int, default=16)
    ap.add_argument("--net-mode", default="tc_tf32x3",
                    help="tc_tf32x3 (default, the bench's) or simt_f64 (the reference's float64 arithmetic)")
    a = ap.parse_args()
    from paper_2409_16504_b200 import sparsenet
    sparsenet.set_mode(a.net_mode)
    w = netplan.init_random(netplan.NetworkPlan(), 0)
    what = {
        "tc_tf32x3": "Full-frame parity of the fused GPU frame (sfb_frame, what bench.py times) vs the CPU "
                     "oracle, every BASELINE config, default network mode tc_tf32x3 (tools/parity_report.py, "
                     "tests/parity_util.py). order/rects/offsets: fused rank order and per-rank tile ranges vs "
                     "the oracle's _prepare/bin_tiles on the same Gaussians; renderer: planes vs the oracle "
                     "renderer on the same Gaussians; e2e: GPU cloud->planes vs oracle cloud->planes; "
                     "e2e_over_pixels: every end-to-end pixel over 2e-3 classified by replaying both blend "
                     "sequences.",
        "simt_f64": "Full-frame parity of the fused GPU frame vs the CPU oracle in the float64 network mode "
                    "(SFB_NET_SIMT_F64, the reference's own arithmetic) (tools/parity_report.py --net-mode "
                    "simt_f64).",
    }.get(a.net_mode, a.net_mode)
    rep = {"what": what, "net_mode": a.net_mode, "tolerance": 2e-3, "frames": {}}
    cloud, views = scenes.config1()
    rep["frames"]["c1"] = run(cloud, views, w, range(len(views)), "c1")
    cloud, views = scenes.config2()
    rep["frames"]["c2"] = run(cloud, views, w, range(len(views)), "c2")
    cloud, views = scenes.config3()
    rep["frames"]["c3"] = run(cloud, views, w, range(min(a.c3_views, len(views))), "c3")
    c4 = []
    for f in range(a.c4_frames):
        cloud, views = scenes.config4_frame(f)
        r = run(cloud, views, w, (0,), f"c4 frame {f}", levels_for=())
        r[0]["frame"] = f
        c4 += r
    rep["frames"]["c4"] = c4
    cloud, views = scenes.config5()
    rep["frames"]["c5"] = run(cloud, views, w, range(min(a.c5_views, len(views))), "c5",
                               levels_for=(0,))
    summ = {}
    for name, recs in rep["frames"].items():
        summ[name] = {
            "frames": len(recs),
            "order_exact": all(r["order"]["order_exact"] for r in recs),
            "rects_offsets_exact": all(r["order"]["rects_exact"] and r["order"]["offsets_exact"]
                                       for r in recs),
            "levels_exact": all(r["levels"]["exact"] for r in recs if "levels" in r),
            "renderer_max_abs": max(s["max_abs"] for r in recs for s in r["renderer"].values()),
            "renderer_over": sum(s["over"] for r in recs for s in r["renderer"].values()),
            "e2e_max_abs": max(s["max_abs"] for r in recs for s in r["e2e"].values()),
            "e2e_over": sum(s["over"] for r in recs for s in r["e2e"].values()),
        }
    rep["summary"] = summ
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(rep, indent=1))
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
