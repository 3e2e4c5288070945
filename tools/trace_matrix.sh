#!/bin/bash
# in-step launch timelines for GPT-J at B = 1/8/16, fp16 and int8
for dt in fp16 int8; do for b in 1 8 16; do
  python tools/launch_trace.py gptj-6b $dt $b | grep -vE "^sum"
done; done
