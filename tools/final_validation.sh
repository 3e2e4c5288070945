#!/bin/bash
# Round-end validation on one B200: GPU tests, smoke, bench lines, BASELINE parity suite, launch lists.
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 700 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo rc=$? >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 500 python bench.py > $O/bench_default.log 2>&1
timeout 300 python bench.py --dtype int8 --no-sweep --no-tp-slices > $O/bench_int8.log 2>&1
for c in gpt2-1.5b gpt-neox-20b; do for d in fp16 int8; do
  timeout 300 python bench.py --config $c --dtype $d --no-sweep --no-tp-slices --no-cpu-baseline > $O/bench_${c}_${d}.log 2>&1
done; done
timeout 900 python tools/parity_baseline.py --suite all --out $O/parity_baseline.json > $O/parity_baseline.log 2>&1; echo parity rc=$? >> $O/parity_baseline.log
for d in fp16 int8; do
  PROF_ACT=auto timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_gptj_${d}_b1.csv python tools/prof_step.py gptj-6b $d 1 0 > $O/ncu_l_$d.log 2>&1
done
