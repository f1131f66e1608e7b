#!/bin/bash
O=gpurun_out/ls.jsonl; : > $O
for cd in "cfg1 f32" "cfg1 bf16" "cfg3 bf16" "cfg3 f32"; do
  set -- $cd
  for LS in 2 3 4; do
    for N in -1 30 48; do
      if [ $N = -1 ]; then unset CKRL_LOSS_CTAS; else export CKRL_LOSS_CTAS=$N; fi
      r=$(timeout 300 python bench.py --config $1 --dtype $2 --loss-streams $LS --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(json.dumps({'ms':round(d['ms_per_step']*1e3,2),'frac':round(r['frac'],3)}))")
      echo "{\"ls\": $LS, \"ctas\": $N, \"cfg\": \"$1\", \"dt\": \"$2\", \"r\": $r}" >> $O
    done
  done
done
