#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_small.py
# (compute-sanitizer was closed on the GPU pool at the end of round 2: the extended workload ran
# without it, rc 0; profiles/r2_sanitizer.summary.txt is the earlier round-2 run)
O=gpurun_out/san; mkdir -p $O; : > $O/summary.txt
for tool in memcheck racecheck synccheck; do
  echo "compute-sanitizer --tool $tool python tools/sanitize_small.py (decode graph off, prefill, int8 W8A8/W8A16/K-group/AUTO B=16, TP-local, full attention stages, QKV attention tail, tensor-core attention, drop-in GEMMs)" >> $O/summary.txt
  timeout 1500 compute-sanitizer --tool $tool python tools/sanitize_small.py > $O/$tool.log 2>&1
  rc=$?
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize workload ok" $O/$tool.log | tail -2 >> $O/summary.txt
  echo "rc=$rc" >> $O/summary.txt
done
