#!/bin/bash
# Round-2 ncu captures (run under gpurun from the repo root): launch list of the headline step
# and --set full captures of every hot kernel. Summarise here with profiles/summarize_ncu.py.
set -x
O=gpurun_out/r2
mkdir -p $O
B="python bench.py --profile --steps 4 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 6 -c 12 --csv --log-file $O/launches_cfg3.csv $B --config cfg3 > $O/l.log 2>&1
for c in cfg3 cfg4 cfg2 cfg1; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tma_tile -s 3 -c 1 \
      -o $O/full_${c}_f32 $B --config $c > $O/f_$c.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tma_tile -s 3 -c 1 \
    -o $O/full_cfg4_bf16 $B --config cfg4 --dtype bf16 > $O/f_cfg4b.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:logits_grad -s 2 -c 1 \
    -o $O/full_grad_cfg4_f32 $B --config cfg4 --grad > $O/f_grad.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:adam -s 6 -c 2 \
    -o $O/full_adam python bench.py --config adam --steps 3 --warmup 3 --adam-params 16777216 > $O/f_adam.log 2>&1
ls -la $O
# keep the box's gpurun_out/ under 64 MiB: raw-page CSVs for every capture, one .ncu-rep kept
for r in $O/full_*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > ${r%.ncu-rep}.details.csv 2>/dev/null
  case $r in *full_cfg3_f32*) ;; *) rm -f $r ;; esac
done
du -sh $O
