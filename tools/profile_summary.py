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
