"""Join an ncu SASS source page (per-instruction stall samples) with nvdisasm -g line info:
stall samples aggregated per CUDA source line, for one kernel.
usage: ncu_lines.py <ncu-rep> <cubin> <mangled kernel name> [top]"""
import csv, io, re, subprocess, sys
from collections import defaultdict

rep, cubin, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
lines = sass.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(f".text.{kern}:"))
where, off2line = "?", {}
for l in lines[start + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        where = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?)\s*;", l)
    if m:
        off2line[int(m.group(1), 16)] = (where, m.group(2))
csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(csvtxt)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ia, iss = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
reasons = [j for j, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][ia], 16)
agg = defaultdict(lambda: [0.0, defaultdict(float), 0])
for r in data:
    off = int(r[ia], 16) - base
    w, ins = off2line.get(off, ("?", r[1].strip()))
    a = agg[w]
    a[0] += float(r[iss] or 0)
    a[2] += 1
    for j in reasons:
        a[1][hdr[j][6:]] += float(r[j] or 0)
tot = sum(a[0] for a in agg.values())
print(f"total stall samples {tot:.0f}")
for w, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    rs = sorted(a[1].items(), key=lambda kv: -kv[1])[:3]
    print(f"{a[0] / tot * 100:5.1f}%  {w:28s} n={a[2]:4d}  " + " ".join(f"{k}={v / max(a[0], 1) * 100:.0f}%" for k, v in rs))
