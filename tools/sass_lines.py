"""Per-source-line stall samples / instructions of one kernel from an ncu SASS
source page (csv) + nvdisasm -g of the same cubin.
usage: python tools/sass_lines.py <ncu sass csv> <nvdisasm -g output> <mangled name> [top]"""
import csv, re, sys, collections
sass_csv, dis, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
data = []
for r in rows[2:]:   # first kernel of the page only
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        data.append(r)
iA, iS, iW, iE = (hdr.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                         "Instructions Executed"))
base = int(data[0][iA], 16)
# offset -> line from nvdisasm
lines = {}
cur_line = None
inside = False
for l in open(dis):
    if l.startswith('\t.section\t.text.'):
        inside = l.strip().endswith(fn) or ('.text.' + fn) in l
        continue
    if not inside:
        continue
    m = re.search(r'line (\d+)', l)
    if '//##' in l and m:
        cur_line = int(m.group(1))
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', l)
    if m:
        lines[int(m.group(1), 16)] = cur_line
agg = collections.defaultdict(lambda: [0.0, 0.0])
tot = [0.0, 0.0]
for r in data:
    off = int(r[iA], 16) - base
    ln = lines.get(off)
    s, e = float(r[iW] or 0), float(r[iE] or 0)
    agg[ln][0] += s
    agg[ln][1] += e
    tot[0] += s
    tot[1] += e
print(f"total stall samples {tot[0]:.0f}, warp instructions {tot[1]:.3g}")
import os
key = 1 if os.environ.get("BY") == "instr" else 0
for ln, (s, e) in sorted(agg.items(), key=lambda x: -x[1][key])[:top]:
    print(f"line {ln}: stall {100*s/tot[0]:5.1f}%  instr {100*e/tot[1]:5.1f}%")
