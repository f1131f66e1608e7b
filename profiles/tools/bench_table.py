"""Markdown table of a bench sweep (profiles/bench_r2.jsonl): one row per JSON line."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
print("| line | dtype | value (env-steps/s) | step µs | dominant kernel | kernel frac | step frac | e2e | CPU baseline |")
print("|---|---|---|---|---|---|---|---|---|")
for d in rows:
    c = d.get("config", {})
    name = c.get("workload", "?").split(":")[0]
    if d.get("impl") == "reference":
        name += " (reference arm)"
    extra = []
    if "head_hidden" in c:
        extra.append(f"head H={c['head_hidden']}")
    if c.get("step_includes", "").startswith("assemble + loss + dlogits"):
        extra.append("+dlogits")
    if extra:
        name += " " + ", ".join(extra)
    r = d.get("roofline") or {}
    kf = r.get("frac")
    sf = r.get("step_frac")
    e2e = (d.get("e2e") or {}).get("value")
    cpu = d.get("cpu_baseline") or {}
    kname = (r.get("kernel") or "").split(" (")[0]
    unit = r.get("unit", "")
    print(f"| {name} | {d.get('dtype')} | {d['value']:.3g} | {d['ms_per_step'] * 1e3:.1f} | {kname} "
          f"| {'' if kf is None else f'{kf:.2f} ({unit})'} | {'' if sf is None else f'{sf:.2f}'} "
          f"| {'' if e2e is None else f'{e2e:.3g}'} | {'' if cpu.get('value') is None else f'{cpu['value']:.3g} ({cpu.get('cores')} thr)'} |")
