"""Summarise one GPU round's ncu outputs into profiles/ (tracked).

usage: python tools/profile_summary.py <tag> [kernel-regex-name]
reads  gpurun_out/launches_<tag>.csv   (ncu --metrics gpu__time_duration.sum launch list)
       gpurun_out/prof_comp_<tag>.ncu-rep (ncu --set full of k_composite)
writes profiles/<tag>_launches.txt, profiles/<tag>_composite_ncu.txt,
       profiles/traffic.json (dram bytes per launch, read by bench.py)
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
tag = sys.argv[1]
out = ROOT / "profiles"
out.mkdir(exist_ok=True)
go = ROOT / "gpurun_out"

# ---- launch list
lp = go / f"launches_{tag}.csv"
if lp.exists():
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "launches.py"), str(lp), "200"],
                       capture_output=True, text=True, check=True)
    (out / f"{tag}_launches.txt").write_text(
        f"# ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none (L2 warm as in the frame, launches serialised)\n"
        f"# one full config-2 frame (the launches between two k_composite), us per kernel name\n"
        + r.stdout)
    print(r.stdout)

# ---- SM-active cycles per kernel (what each kernel costs the concurrent lanes)
sp = go / f"smlaunch_{tag}.csv"
if sp.exists():
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "smcost.py"), str(sp)],
                       capture_output=True, text=True, check=True)
    (out / f"{tag}_smcost.txt").write_text(
        "# ncu sm__cycles_active.sum per kernel of one config-2 frame (launches serialised, L2 warm)\n"
        + r.stdout)
    print(r.stdout)

# ---- full capture of the compositor
rep = go / f"prof_comp_{tag}.ncu-rep"
if rep.exists():
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]
    vals = {}
    lines = []
    for k in want:
        if k in h:
            i = h.index(k)
            vals[k] = (v[i], u[i])
            lines.append(f"{k:70s} {v[i]} {u[i]}")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(vals["dram__bytes_read.sum"][0]) * scale[vals["dram__bytes_read.sum"][1]]
    wr = float(vals["dram__bytes_write.sum"][0]) * scale[vals["dram__bytes_write.sum"][1]]
    txt = (f"# ncu --set full --clock-control none of k_composite (config-2 frame), tag {tag}\n"
           + "\n".join(lines) + f"\nDRAM bytes per launch (read+write): {rd + wr:.0f}\n")
    (out / f"{tag}_composite_ncu.txt").write_text(txt)
    print(txt)
    tj = out / "traffic.json"
    d = json.loads(tj.read_text()) if tj.exists() else {}
    d["k_composite"] = {"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr,
                        "source": f"profiles/{tag}_composite_ncu.txt"}
    tj.write_text(json.dumps(d, indent=1) + "\n")

# ---- tcgen05 conv launches (tools/conv_profile.sh): the last frame's convs
cp = go / f"conv_ncu_{tag}.csv"
if cp.exists():
    rows = [r for r in csv.reader(open(cp)) if len(r) > 10]
    h = rows[0]
    ix = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Grid Size")}
    per = {}
    for r in rows[1:]:
        d = per.setdefault(int(r[ix["ID"]]), {"k": r[ix["Kernel Name"]], "grid": r[ix["Grid Size"]]})
        d[r[ix["Metric Name"]]] = r[ix["Metric Value"]]
    ids = sorted(per)
    starts = [i for i in ids if per[i]["k"].startswith("void k_conv_narrow")]
    # a complete frame: from the second-to-last level-0 conv to the last
    # (the launch cap may cut the last frame short)
    last = ([i for i in ids if starts[-2] <= i < starts[-1]] if len(starts) >= 2
            else [i for i in ids if i >= starts[-1]] if starts else ids)
    f = lambda d, m: float(d.get(m, "0").replace(",", "") or 0)
    lines = [f"# ncu of the convolution launches of one steady-state config-2 frame (view 0), tag {tag}",
             "# (tools/conv_profile.sh: --clock-control none --cache-control none, launches serialised, lanes 1)",
             "# tensor% = sm__pipe_tensor_cycles_active (avg over SMs / busiest SM), tmem = smsp__inst_executed_pipe_tmem.sum,",
             "# warps% = sm__warps_active; smem-occ = CTAs per SM allowed by shared memory",
             f"{'kernel':34s} {'grid':>6s} {'us':>6s} {'tensor% avg':>11s} {'max':>6s} {'tmem inst':>9s} {'DRAM MB':>8s} {'warps%':>6s} {'smem-occ':>8s} {'cluster':>7s}"]
    for i in last:
        d = per[i]
        name = d["k"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[:34]
        lines.append(f"{name:34s} {d['grid'].strip('()').split(',')[0]:>6s} {f(d, 'gpu__time_duration.sum') / 1000:6.1f} "
                     f"{f(d, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):11.2f} "
                     f"{f(d, 'sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_active'):6.1f} "
                     f"{f(d, 'smsp__inst_executed_pipe_tmem.sum'):9.0f} "
                     f"{(f(d, 'dram__bytes_read.sum') + f(d, 'dram__bytes_write.sum')) / 1e6:8.2f} "
                     f"{f(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} "
                     f"{f(d, 'launch__occupancy_limit_shared_mem'):8.0f} {f(d, 'launch__cluster_dim_x'):7.0f}")
    (out / f"{tag}_conv_ncu.txt").write_text("\n".join(lines) + "\n")

# ---- every launch of one frame in issue order (from the SM-cost capture)
sp = go / f"smlaunch_{tag}.csv"
if sp.exists():
    rows = [r for r in csv.reader(open(sp)) if len(r) > 10]
    h = rows[0]
    ix = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Grid Size", "Block Size")}
    per = {}
    for r in rows[1:]:
        d = per.setdefault(int(r[ix["ID"]]), {"k": r[ix["Kernel Name"]], "g": r[ix["Grid Size"]],
                                              "b": r[ix["Block Size"]]})
        d[r[ix["Metric Name"]]] = r[ix["Metric Value"]]
    ids = sorted(per)
    starts = [i for i in ids if "k_bbox_init" in per[i]["k"]]
    if len(starts) >= 2:
        a, b = starts[-2], starts[-1]
        fr = [i for i in ids if a <= i < b]
        num = lambda d, m: float(d.get(m, "0").replace(",", "") or 0)
        tot = sum(num(per[i], "gpu__time_duration.sum") / 1000 for i in fr)
        lines = ["# every kernel launch of one config-2 frame (view 0), in issue order: ncu --metrics gpu__time_duration.sum,",
                 "# sm__cycles_active.sum,sm__warps_active --clock-control none --cache-control none (launches serialised;",
                 "# per-launch times are cold-start + serialised, so compare SHARES, not absolutes, with bench.py's timings)",
                 f"# tag {tag}, command: python bench.py --steps 2 --warmup 1 --lanes 1 --no-e2e --no-cpu --no-profile --view 0",
                 f"{'#':>3s} {'us':>7s} {'share%':>6s} {'grid':>6s} {'block':>5s} {'warps%':>6s}  kernel"]
        for n, i in enumerate(fr):
            d = per[i]
            t = num(d, "gpu__time_duration.sum") / 1000
            name = d["k"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
            lines.append(f"{n:3d} {t:7.1f} {100 * t / tot:6.1f} {d['g'].strip('()').split(',')[0]:>6s} "
                         f"{d['b'].strip('()').split(',')[0]:>5s} "
                         f"{num(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f}  {name}")
        lines.append(f"total {tot:.1f} us serialised over {len(fr)} launches")
        (out / f"{tag}_launches.txt").write_text("\n".join(lines) + "\n")
