# A/B: default libckrl.so vs an alternative build $1, interleaved, configs in $2..
alt=$1; shift
for c in "$@"; do for i in 1 2 3; do for lib in paper_2510_06710_b200/libckrl.so $alt; do CKRL_LIB=$PWD/$lib timeout 300 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(\"$lib $c\", round(j[\"value\"]/1e6,2), 'step', round(j[\"ms_per_step\"]*1e3,1), 'kern', round(j[\"roofline\"][\"kernel_ms\"]*1e3,1))"; done; done; done
