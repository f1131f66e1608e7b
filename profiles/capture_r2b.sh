#!/bin/bash
# Round-2 (second half) captures, run under gpurun from the repo root: launch lists of the
# chained cfg3 step, the policy-head step (--head 4096) and one cfg5 epoch, plus a --set full
# capture of the tcgen05 projection kernel. Summarised in profiles/ncu_r2b.md.
O=gpurun_out/r2b
mkdir -p $O
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
B="python bench.py --profile --steps 4 --warmup 3 --no-cpu-baseline"
timeout 600 ncu $M -c 40 --log-file $O/launches_cfg3.csv $B --config cfg3 > $O/l3.log 2>&1
timeout 600 ncu $M -k regex:'proj_stats|tile_kernel|assemble' -c 30 --log-file $O/launches_head4096.csv $B --config cfg3 --head 4096 > $O/lh.log 2>&1
timeout 600 ncu $M -k regex:'gen_kernel|env_chunk|act_scatter|boot_kernel|episodes_kernel' -c 60 --log-file $O/launches_cfg5.csv \
    python bench.py --config cfg5 --steps 1 --warmup 3 --stages 1 --placements colocated --samplers parallel > $O/l5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:proj_stats -s 2 -c 1 -o $O/full_proj4096 \
    python profiles/tools/proj_once.py 4096 > $O/fp.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:proj_stats -s 2 -c 1 -o $O/full_proj1024 \
    python profiles/tools/proj_once.py 1024 > $O/fp1.log 2>&1
for r in $O/full_*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > ${r%.ncu-rep}.details.csv 2>/dev/null
done
ls -la $O
