#!/bin/bash
# B=1 plan / PDL sweep: tools/xs_sweep.sh [fp16|int8] [B]
dt=${1:-fp16}; b=${2:-1}
for xs in 0 1; do for mask in 0x04 0x84 0x8d 0xbd 0xff; do
  echo "== XS=$xs PDL=$mask"; DSINF_XS=$xs DSINF_PDL_MASK=$mask python tools/launch_trace.py gptj-6b $dt $b | head -1
done; done
