#!/bin/bash
# persistent-kernel parameter sweep (device-timed decode ms/step)
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step'],4), d['roofline']['step']['frac'])"; }
run() { env "$@" python bench.py --steps 32 --warmup 4 --no-cpu-baseline --no-pdl $EXTRA 2>&1 | summ "$*"; }
run DSINF_STEP_CS=2
run DSINF_STEP_CS=4
run DSINF_STEP_CS=8
run DSINF_STEP_CS=4 DSINF_STEP_LA=4
run DSINF_STEP_CS=4 DSINF_STEP_STAGES=6
