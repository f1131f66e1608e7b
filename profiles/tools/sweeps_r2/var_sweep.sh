#!/bin/bash
O=gpurun_out/var.jsonl; : > $O
for V in 4 0 3; do
  for cd in "cfg4 bf16" "cfg3 bf16" "cfg2 bf16" "cfg4 f32"; do
    set -- $cd
    r=$(CKRL_TMA_VARIANT=$V timeout 300 python bench.py --config $1 --dtype $2 --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(json.dumps({'ms':round(d['ms_per_step']*1e3,2),'frac':round(r['frac'],3),'alone':round(r.get('frac_alone') or 0,3)}))")
    echo "{\"var\": $V, \"cfg\": \"$1\", \"dt\": \"$2\", \"r\": $r}" >> $O
  done
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/intree_tests.log 2>&1; echo rc=$? >> gpurun_out/intree_tests.log
