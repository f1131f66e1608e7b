"""Per-kernel HBM table from ncu launch lists (every kernel's achieved GB/s from
`dram__bytes_{read,write}.sum` / `gpu__time_duration.sum`, against the measured copy bandwidth and
the north star's nominal 8 TB/s).

usage: kernel_table.py <peak GB/s> <label>=<launches.csv> ...

ncu serialises launches and runs each one cold, so these are per-launch figures of a kernel
running alone — the bench's in-pipeline numbers are the ones the step sees."""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(.*$", "", name) if not name.startswith("void ") else name[5:]
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("ckrl::", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    return name.strip()


def load(path):
    rows = [l for l in open(path) if l.startswith('"')]
    recs = collections.defaultdict(dict)
    for r in csv.DictReader(rows):
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3,
                 "nsecond": 1, "ms": 1e6, "msecond": 1e6}.get(u, 1)
        recs[(r["ID"], r["Kernel Name"])][r["Metric Name"]] = v * scale
    return recs


def main():
    peak = float(sys.argv[1])
    print("| workload | kernel | launches | µs / launch | MB / launch | GB/s | of measured | of 8 TB/s |")
    print("|---|---|---|---|---|---|---|---|")
    for arg in sys.argv[2:]:
        label, path = arg.split("=", 1)
        agg = collections.OrderedDict()
        for (_, kname), m in load(path).items():
            k = short(kname)
            if k.startswith("at::") or "elementwise" in k or "distribution" in k:
                continue
            t = m.get("gpu__time_duration.sum", 0.0)
            b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
            a = agg.setdefault(k, [0, 0.0, 0.0])
            a[0] += 1
            a[1] += t
            a[2] += b
        for k, (n, t, b) in agg.items():
            us, mb = t / n / 1e3, b / n / 1e6
            gbs = b / t if t else 0.0
            print(f"| {label} | `{k}` | {n} | {us:.1f} | {mb:.2f} | {gbs:.0f} | {gbs / peak:.2f} | {gbs / 8000:.2f} |")


if __name__ == "__main__":
    main()
