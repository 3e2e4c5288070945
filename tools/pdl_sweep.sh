#!/bin/bash
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step'],4))"; }
for m in 0x7f 0x00 0x04 0x06 0x02 0x40 0x3b 0x01 0x08 0x10 0x20; do
  DSINF_PDL_MASK=$m python bench.py --steps 32 --warmup 4 --no-cpu-baseline "$@" 2>&1 | summ mask=$m
done
