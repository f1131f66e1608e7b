#!/bin/bash
# Round-1 measurement sweep (run under gpurun from the repo root): every config x dtype, the
# f1 (logits gradient) and f4 (Adam) lines and the cfg5 pipeline, one JSON line each.
O=gpurun_out/bench_r1.jsonl
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
timeout 300 python bench.py --config adam --steps 20 >> $O 2>/dev/null
timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 >> $O 2>/dev/null
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 >> $O 2>/dev/null
wc -l $O
