#!/bin/bash
# stages x CTA-per-SM cap x PDL mask: tools/occ_sweep.sh [fp16|int8] [B]
dt=${1:-fp16}; b=${2:-1}
for st in 2 3 4; do for cap in 0 2; do for mask in 0x8d 0xff; do
  r=$(DSINF_STAGES=$st DSINF_CTA_PER_SM=$cap DSINF_PDL_MASK=$mask python tools/launch_trace.py gptj-6b $dt $b 2>&1 | grep step)
  echo "st=$st cap=$cap pdl=$mask $r"
done; done; done
