"""Per-source-line stall samples of one kernel from an ncu source page (SASS) export.

usage: sass_lines.py <sass.csv from `ncu -i R --page source --csv --print-source sass`>
                     <nvdisasm -g -c output of the same cubin> <mangled kernel name> [top]
Maps each sampled SASS offset to its -lineinfo source line and prints samples, executed
warp instructions and the top stall reasons per line."""
import collections
import csv
import re
import sys

sass_csv, dis, K = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = open(dis).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + K + ":"))
fnline = re.compile(r'//## File "([^"]+)", line (\d+)')
ins = re.compile(r"/\*([0-9a-f]{4,})\*/")
off2line, cur = {}, None
for l in lines[start + 1:]:
    if l.startswith(".text."):
        break
    m = fnline.search(l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = ins.search(l)
    if m:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
h, data = rows[1], rows[2:]
ia, isamp, iex = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stalls = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
base = int(data[0][ia], 16)
agg, aex = collections.Counter(), collections.Counter()
rs = collections.defaultdict(collections.Counter)
for r in data:
    ln = off2line.get(int(r[ia], 16) - base)
    agg[ln] += int(r[isamp])
    aex[ln] += int(r[iex])
    for i in stalls:
        rs[ln][h[i][6:]] += int(r[i] or 0)
tot = sum(agg.values())
print(f"total samples {tot}")
for ln, s in agg.most_common(top):
    why = ", ".join(f"{k} {v}" for k, v in rs[ln].most_common(3) if v)
    print(f"{s:6d} {100 * s / tot:5.1f}% exec {aex[ln]:9d}  {ln}  [{why}]")
