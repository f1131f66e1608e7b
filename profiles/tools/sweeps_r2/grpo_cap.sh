#!/bin/bash
O=gpurun_out/grpo_cap.jsonl; : > $O
run() {
  if [ $3 = -1 ]; then unset CKRL_LOSS_CTAS; else export CKRL_LOSS_CTAS=$3; fi
  r=$(timeout 300 python bench.py --config $1 --dtype $2 --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(json.dumps({'ms':round(d['ms_per_step']*1e3,2),'frac':round(r['frac'],3)}))")
  echo "{\"ctas\": $3, \"cfg\": \"$1\", \"dt\": \"$2\", \"r\": $r}" >> $O
}
for rep in 1 2; do
for N in -1 40 49 56 64; do run cfg2 bf16 $N; done
for N in -1 88 120; do run cfg2 f32 $N; done
done
