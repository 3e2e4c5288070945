#!/bin/bash
# quick decode timing variants: tools/bench_quick.sh [extra bench args...]
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step'],4), 'ms', d['roofline']['step']['frac'] if d.get('roofline') else '')"; }
python bench.py --steps 32 --warmup 4 --no-cpu-baseline "$@" 2>&1 | summ pdl
python bench.py --steps 32 --warmup 4 --no-cpu-baseline --no-pdl "$@" 2>&1 | summ nopdl
