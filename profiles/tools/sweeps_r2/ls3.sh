#!/bin/bash
O=gpurun_out/ls3.jsonl; : > $O
for rep in 1 2; do
for cd in "cfg3 f32" "cfg3 bf16" "cfg1 f32" "cfg1 bf16" "cfg2 f32" "cfg2 bf16"; do
  set -- $cd
  for LS in 2 3; do
    r=$(timeout 300 python bench.py --config $1 --dtype $2 --loss-streams $LS --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(json.dumps({'ms':round(d['ms_per_step']*1e3,2),'frac':round(r['frac'],3)}))")
    echo "{\"ls\": $LS, \"cfg\": \"$1\", \"dt\": \"$2\", \"r\": $r}" >> $O
  done
done
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ls3_tests.log 2>&1; echo rc=$? >> gpurun_out/ls3_tests.log
timeout 300 python bench.py > gpurun_out/ls3_default.json 2>/dev/null
