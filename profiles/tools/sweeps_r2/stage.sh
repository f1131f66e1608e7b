#!/bin/bash
O=gpurun_out/stage.jsonl; : > $O
for c in cfg1 cfg3; do
for KB in 40 56 72; do for NS in 2 3; do
  r=$(CKRL_STAGE_KB=$KB CKRL_NSTAGE=$NS timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(json.dumps({'ms':round(d['ms_per_step']*1e3,2),'frac':round(r['frac'],3)}))")
  echo "{\"cfg\": \"$c\", \"kb\": $KB, \"ns\": $NS, \"r\": $r}" >> $O
done; done; done
