#!/bin/bash
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step'],4))"; }
for i in 1 2; do
python bench.py --steps 32 --warmup 4 --no-cpu-baseline --no-pdl "$@" 2>&1 | summ nopdl
python bench.py --steps 32 --warmup 4 --no-cpu-baseline "$@" 2>&1 | summ pdl
DSINF_PDL_MASK=0 python bench.py --steps 32 --warmup 4 --no-cpu-baseline "$@" 2>&1 | summ mask0
done
