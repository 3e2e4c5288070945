summ() { python -c "import json,sys; d=json.loads([l for l in sys.stdin.read().splitlines() if l.startswith('{')][-1]); k=d['roofline']['in_step_interval']['kinds']; print('$1', round(d['ms_per_step'],4), {n:v['interval_us_mean'] for n,v in k.items()})"; }
B="timeout 200 python bench.py --steps 32 --warmup 4 --no-cpu-baseline --no-sweep --no-tp-slices"
for a in "--dtype int8" "--dtype fp16" "--dtype int8 --batch 16" "--dtype fp16 --batch 16" "--dtype int8 --batch 8"; do $B $a 2>&1 | summ "default $a"; done
for r in 3 4; do DSINF_ATTN_RING=$r $B --dtype int8 --batch 16 2>&1 | summ "ring=$r int8 b16"; done
for c in 1024 2048; do DSINF_ATTN_CTAS=$c $B --dtype int8 --batch 16 2>&1 | summ "ctas=$c int8 b16"; done
DSINF_ATTN_CTAS=1024 DSINF_ATTN_RING=4 $B --dtype int8 --batch 16 2>&1 | summ "ctas=1024 ring4 int8 b16"
for r in 3 4; do DSINF_ATTN_RING=$r $B --dtype int8 2>&1 | summ "ring=$r int8 b1"; done
