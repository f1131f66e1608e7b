#!/bin/bash
# Per-kernel HBM table (achieved GB/s of every kernel from ncu dram bytes / duration):
# launch lists of the cfg3 / cfg2 / cfg4 steps (f32 and bf16), the policy-head step, one cfg5
# epoch, the standalone dlogits kernel and Adam. Summarised by profiles/tools/kernel_table.py
# into DESIGN §6.
O=gpurun_out/kt
mkdir -p $O
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
B="python bench.py --profile --steps 4 --warmup 3 --no-cpu-baseline"
K='regex:ckrl|tile_kernel|assemble|grpo|proj|adam|gen_kernel|env_chunk|act_scatter|boot|episodes|logits_grad|gae'
for c in cfg3 cfg2 cfg4 cfg1; do
  timeout 600 ncu $M -k $K -c 40 --log-file $O/launches_${c}_f32.csv $B --config $c > $O/l_$c.log 2>&1
done
for c in cfg3 cfg4; do
  timeout 600 ncu $M -k $K -c 40 --log-file $O/launches_${c}_bf16.csv $B --config $c --dtype bf16 > $O/lb_$c.log 2>&1
done
timeout 600 ncu $M -k $K -c 30 --log-file $O/launches_head4096.csv $B --config cfg3 --head 4096 > $O/lh.log 2>&1
timeout 600 ncu $M -k $K -c 80 --log-file $O/launches_cfg5.csv \
    python bench.py --config cfg5 --steps 1 --warmup 3 --stages 1 --placements colocated --samplers parallel > $O/l5.log 2>&1
timeout 600 ncu $M -k $K -c 20 --log-file $O/launches_grad.csv $B --config cfg4 --grad separate > $O/lg.log 2>&1
timeout 600 ncu $M -k $K -c 12 --log-file $O/launches_adam.csv \
    python bench.py --config adam --steps 3 --warmup 3 > $O/la.log 2>&1
ls -la $O
