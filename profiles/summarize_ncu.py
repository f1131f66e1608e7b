"""Summarise ncu captures (run here, on the CPU box) into profiles/ncu_<tag>.md + ncu_traffic.json.

    python profiles/summarize_ncu.py <tag> <launches.csv> <full_*.raw.csv | full_*.ncu-rep> ...

Inputs are what profiles/capture_r1.sh leaves in gpurun_out/r1/: the launch list of the
headline step (gpu__time_duration / dram bytes per launch) and `--page raw --csv` exports of
`--set full` captures (a .ncu-rep is exported here). Every kernel row of every capture gets a
table; DRAM traffic per launch (read + write) of the loss kernel captures goes to
ncu_traffic.json, keyed "<cfg>_<dtype>", where bench.py reads its roofline.traffic.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "smsp__warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__warps_issue_stalled_mio_throttle_per_issue_active.ratio"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def launches(path):
    out, hdr = [], None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.append((d["ID"], d["Kernel Name"].split("(")[0], d["Metric Name"], d["Metric Value"],
                        d.get("Metric Unit", "")))
    return out


def raw_rows(path):
    if path.endswith(".ncu-rep"):
        text = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    else:
        text = open(path).read()
    r = list(csv.reader(io.StringIO(text)))
    hdr, units = r[0], r[1]
    return [(dict(zip(hdr, row)), dict(zip(hdr, units))) for row in r[2:] if len(row) == len(hdr)]


def num(vals, units, k):
    v = float(vals.get(k, "0").replace(",", "") or 0)
    return v * SCALE.get(units.get(k, ""), 1)


def main():
    tag, lcsv, caps = sys.argv[1], sys.argv[2], sys.argv[3:]
    md = [f"# ncu summary — {tag}", "",
          "Launch list of the headline step (`bench.py --config cfg3 --profile`: assemble + fused loss per "
          "step; ncu serialises and cold-starts each launch, so compare shares, not absolutes).", "",
          "| id | kernel | metric | value | unit |", "|---|---|---|---|---|"]
    for i, k, m, v, u in launches(lcsv):
        md.append(f"| {i} | `{k}` | {m} | {v} | {u} |")
    traffic = {}
    for path in caps:
        name = re.sub(r"\.(raw\.csv|ncu-rep)$", "", os.path.basename(path))
        for idx, (vals, units) in enumerate(raw_rows(path)):
            kname = vals.get("Kernel Name", "?").split("(")[0]
            md += ["", f"## `{name}` launch {idx}: `{kname}` (--set full)", "", "| metric | value | unit |",
                   "|---|---|---|"]
            for k in KEYS:
                if k in vals:
                    md.append(f"| {k} | {vals[k]} | {units.get(k, '')} |")
            t_us = num(vals, units, "gpu__time_duration.sum")
            rw = num(vals, units, "dram__bytes_read.sum") + num(vals, units, "dram__bytes_write.sum")
            if t_us > 0:
                md.append(f"| (derived) DRAM GB/s | {rw / (t_us * 1e-6) / 1e9:.1f} | GB/s |")
            m = re.match(r"full_(cfg\d)_(f32|bf16)$", name)
            if m and "tma_tile" in kname:
                traffic[f"{m.group(1)}_{m.group(2)}"] = rw
            if name.startswith("full_grad_"):
                traffic[name[len("full_"):]] = rw
    out = os.path.join(HERE, f"ncu_{tag}.md")
    keep = ""  # hand-written sections (from "## Fused") survive a regeneration
    if os.path.exists(out):
        old_md = open(out).read()
        i = old_md.find("\n## Fused")
        keep = old_md[i:] if i >= 0 else ""
    with open(out, "w") as f:
        f.write("\n".join(md) + "\n" + keep)
    tpath = os.path.join(HERE, "ncu_traffic.json")
    old = json.load(open(tpath)) if os.path.exists(tpath) else {}
    old.update(traffic)
    json.dump(old, open(tpath, "w"), indent=1, sort_keys=True)
    print("\n".join(md[:40]))
    print(json.dumps(old, indent=1))


if __name__ == "__main__":
    main()
