summ() { python -c "import json,sys; d=json.loads([l for l in sys.stdin.read().splitlines() if l.startswith('{')][-1]); k=d['roofline']['in_step_interval']['kinds']; print('$1', round(d['ms_per_step'],4), {n:v['interval_us_mean'] for n,v in k.items()})"; }
B="timeout 200 python bench.py --steps 32 --warmup 4 --no-cpu-baseline --no-sweep --no-tp-slices"
for a in "--dtype int8" "--dtype fp16" "--dtype fp16 --batch 8" "--dtype int8 --batch 2" "--config gpt2-1.5b --dtype fp16" "--config gpt2-1.5b --dtype int8"; do
  for f in 0 1; do DSINF_ATTN_FUSE=$f $B $a 2>&1 | summ "fuse=$f $a"; done
done
