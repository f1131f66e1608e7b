#!/bin/bash
O=gpurun_out/head_ab.jsonl; : > $O
for rep in 1 2 3; do
for L in exp/libckrl_old.so paper_2510_06710_b200/libckrl.so; do
  for h in 1024 4096; do
    r=$(CKRL_LIB=$L timeout 300 python bench.py --config cfg3 --head $h --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(json.dumps({'ms':round(d['ms_per_step']*1e3,2),'kms':round(r['kernel_ms']*1e3,2),'rows':r.get('loss_from_rows_ms_alone')}))")
    echo "{\"lib\": \"$L\", \"h\": $h, \"r\": $r}" >> $O
  done
done
done
