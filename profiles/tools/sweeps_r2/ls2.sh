#!/bin/bash
O=gpurun_out/ls2.jsonl; : > $O
run() { # cfg dt ls ctas
  if [ $4 = -1 ]; then unset CKRL_LOSS_CTAS; else export CKRL_LOSS_CTAS=$4; fi
  r=$(timeout 300 python bench.py --config $1 --dtype $2 --loss-streams $3 --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(json.dumps({'ms':round(d['ms_per_step']*1e3,2),'frac':round(r['frac'],3)}))")
  echo "{\"ls\": $3, \"ctas\": $4, \"cfg\": \"$1\", \"dt\": \"$2\", \"r\": $r}" >> $O
}
for LS in 3 4; do for N in 56 64 74 88 104; do run cfg3 f32 $LS $N; done; done
for LS in 3 4; do for N in 40 48 56 64 74; do run cfg3 bf16 $LS $N; done; done
for LS in 3 4; do for N in -1 74 104 142; do run cfg2 f32 $LS $N; done; done
for LS in 3 4; do for N in -1 74 104; do run cfg2 bf16 $LS $N; done; done
for LS in 2 3; do run cfg4 f32 $LS -1; run cfg4 bf16 $LS -1; done
