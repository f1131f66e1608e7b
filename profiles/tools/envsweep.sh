# envsweep.sh "<ENV=a ENV=b ...>" configs... : each config (cfgN[:bf16]) under each env setting
# (settings separated by spaces, multiple vars in one setting joined with ',')
sets=$1; shift
for cd in "$@"; do c=${cd%%:*}; dt=f32; [ "$c" != "$cd" ] && dt=${cd#*:}; for i in 1 2; do for st in $sets; do env ${st//,/ } timeout 300 python bench.py --config $c --dtype $dt --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(\"$st $cd\", round(j[\"value\"]/1e6,2), 'step', round(j[\"ms_per_step\"]*1e3,1), 'kern', round(j[\"roofline\"][\"kernel_ms\"]*1e3,1))"; done; done; done
