#!/bin/bash
# Step-kernel experiment matrix: env settings x (fp16, int8) at B=1 (tools/step_bench.py).
# usage: tools/sk_matrix.sh "ENV1=a ENV2=b" "ENV1=c" ...
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 300 python tools/step_bench.py ${SKM_CFG:-gptj-6b} ${SKM_DT:-fp16,int8} ${SKM_B:-1} 32 2>&1 | grep -v "^$" | tail -4
done
