#!/bin/bash
# env-knob sweep of the decode step: tools/knob_sweep.sh "<VAR=val ...>" [bench args...]
settings=$1; shift
summ() { python -c "import json,sys; d=json.loads([l for l in sys.stdin.read().splitlines() if l.startswith('{')][-1]); k=d['roofline']['in_step_interval']['kinds']; print('$1', round(d['ms_per_step'],4), {n:v['interval_us_mean'] for n,v in k.items()})"; }
for kv in $settings; do
  env $(echo $kv | tr "," " ") timeout 200 python bench.py --steps 32 --warmup 4 --no-cpu-baseline --no-sweep --no-tp-slices "$@" 2>&1 | summ "$kv $*"
done
