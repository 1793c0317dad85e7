"""Hottest source lines (warp-stall samples) per kernel of an ncu report:
python tools/src_hot.py report.ncu-rep [name-substring] [lines]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
nl = int(sys.argv[3]) if len(sys.argv) > 3 else 10
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Function Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif r and r[0] == "Line No" and cur is not None:
        cur["hdr"] = r
    elif cur is not None and "hdr" in cur:
        cur["rows"].append(r)
seen = set()
for b in blocks:
    if want not in b["name"] or b["name"] in seen:
        continue
    seen.add(b["name"])
    h = b["hdr"]
    i_s = h.index("Warp Stall Sampling (All Samples)")
    recs, tot = [], 0
    for r in b["rows"]:
        if r and r[0]:
            try:
                recs.append((int(r[0]), r[1][:100], int(r[i_s])))
                tot += int(r[i_s])
            except ValueError:
                pass
    if not tot:
        continue
    print(f"== {b['name'][:90]}  ({tot} samples)")
    for line, src, smp in sorted(recs, key=lambda x: -x[2])[:nl]:
        print(f"{line:5d} {100 * smp / tot:5.1f}%  {src}")
