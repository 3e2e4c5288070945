#!/bin/bash
# L2 warm-up sweep: DSINF_NEXT_MASK x DSINF_NEXT_STAGES on the default decode bench
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step'],4), 'ms')"; }
for mask in 0x0 0x1f 0x02 0x1d; do
  for st in -2 2 8; do
    DSINF_NEXT_MASK=$mask DSINF_NEXT_STAGES=$st python bench.py --steps 32 --warmup 4 --no-cpu-baseline "$@" 2>&1 | summ "mask=$mask stages=$st"
  done
done
