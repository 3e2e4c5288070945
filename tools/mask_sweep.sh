#!/bin/bash
# DSINF_PDL_MASK sweep of the decode step (bits: 0 qkv, 1 attention, 2 attn-out, 3 up, 4 down,
# 5 lm head, 6 the rest, 7 row_prep): tools/mask_sweep.sh "<masks>" [bench args...]
masks=$1; shift
summ() { python -c "import json,sys; d=json.loads([l for l in sys.stdin.read().splitlines() if l.startswith('{')][-1]); k=d['roofline']['in_step_interval']['kinds']; print('$1', round(d['ms_per_step'],4), {n:v['interval_us_mean'] for n,v in k.items()})"; }
for m in $masks; do
  DSINF_PDL_MASK=$m timeout 200 python bench.py --steps 32 --warmup 4 --no-cpu-baseline --no-sweep --no-tp-slices "$@" 2>&1 | summ "mask=$m $*"
done
