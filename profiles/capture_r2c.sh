#!/bin/bash
# Round-2 (end) bf16 captures after the per-tile row finish and packed bf16 words: the full
# bench sweep (profiles/bench_all_r2.sh), the cfg4 bf16 launch list and --set full captures of
# the cfg4 / cfg3 bf16 loss kernels. Summarised in profiles/ncu_r2c.md.
bash profiles/bench_all_r2.sh > gpurun_out/sweep.log 2>&1
O=gpurun_out/r2c; mkdir -p $O
B="python bench.py --profile --steps 4 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 6 -c 12 --csv --log-file $O/launches_cfg4_bf16.csv $B --config cfg4 --dtype bf16 > $O/l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tma_tile -s 3 -c 1 \
    -o $O/full_cfg4_bf16 $B --config cfg4 --dtype bf16 > $O/f.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tma_tile -s 3 -c 1 \
    -o $O/full_cfg3_bf16 $B --config cfg3 --dtype bf16 > $O/f3.log 2>&1
for r in $O/full_*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > ${r%.ncu-rep}.details.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > ${r%.ncu-rep}.sass.csv 2>/dev/null
done
