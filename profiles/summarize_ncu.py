"""Summarise ncu captures (run here, on the CPU box) into profiles/*.md + ncu_traffic.json.

    python profiles/summarize_ncu.py <tag> <launches.csv> <full-cfg3.ncu-rep> [<full-cfg4.ncu-rep>]
"""
import csv
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.append((d["ID"], d["Kernel Name"].split("(")[0], d["Metric Name"], d["Metric Value"]))
    return out


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]


def main():
    tag, lcsv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    md = [f"# ncu summary — {tag}", "", "## Launch list (one bench step = assemble + fused loss; ncu serialises and cold-starts each launch)", "",
          "| id | kernel | metric | value |", "|---|---|---|---|"]
    for i, k, m, v in launches(lcsv):
        md.append(f"| {i} | `{k}` | {m} | {v} |")
    traffic = {}
    for rep in reps:
        name = os.path.basename(rep).replace(".ncu-rep", "")
        vals, units = raw(rep)
        md += ["", f"## `{name}` (--set full, 1 launch)", "", "| metric | value | unit |", "|---|---|---|"]
        for k in KEYS:
            if k in vals:
                md.append(f"| {k} | {vals[k]} | {units.get(k, '')} |")
        rd = float(vals.get("dram__bytes_read.sum", "0").replace(",", ""))
        wr = float(vals.get("dram__bytes_write.sum", "0").replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(units.get("dram__bytes_read.sum", "byte"), 1)
        wr *= scale.get(units.get("dram__bytes_write.sum", "byte"), 1)
        cfg = "cfg4" if "cfg4" in name else ("cfg3" if "cfg3" in name else name)
        traffic[f"{cfg}_f32"] = rd + wr
    with open(os.path.join(HERE, f"ncu_{tag}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    tpath = os.path.join(HERE, "ncu_traffic.json")
    old = json.load(open(tpath)) if os.path.exists(tpath) else {}
    old.update(traffic)
    json.dump(old, open(tpath, "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
