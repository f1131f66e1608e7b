#!/bin/bash
# Round-2 measurement sweep (run under gpurun from the repo root): every config x dtype, the
# f1 (logits gradient), f4 (Adam) and N2 (policy head, --head) lines, the cfg5 pipeline
# variants and the reference arm; one JSON line each in gpurun_out/bench_r2.jsonl.
O=gpurun_out/bench_r2.jsonl
: > $O
timeout 600 python bench.py >> $O 2>gpurun_out/bench_default.err
for c in cfg1 cfg2 cfg4; do
  timeout 300 python bench.py --config $c --steps 100 --warmup 5 >> $O 2>/dev/null
done
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 300 python bench.py --config $c --dtype bf16 --steps 100 --warmup 5 --no-cpu-baseline >> $O 2>/dev/null
done
for c in cfg3 cfg4; do
  timeout 300 python bench.py --config $c --grad fused --steps 60 --warmup 5 --no-cpu-baseline >> $O 2>/dev/null
done
for h in 4096 1024; do
  timeout 300 python bench.py --config cfg3 --head $h --steps 60 --warmup 5 >> $O 2>/dev/null
done
timeout 300 python bench.py --config adam --steps 20 >> $O 2>/dev/null
timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 >> $O 2>/dev/null
for c in cfg3 cfg2 cfg4 cfg5; do
  timeout 300 python bench.py --impl reference --config $c --steps 3 --warmup 1 >> $O 2>/dev/null
done
wc -l $O
