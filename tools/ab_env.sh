#!/bin/bash
# A/B an env var on the in-situ launch trace: tools/ab_env.sh VAR "v1 v2 ..." [launch_trace args]
var=$1; vals=$2; shift 2
for v in $vals; do
  echo "== $var=$v"; env $var=$v python tools/launch_trace.py "$@" | grep -vE "^sum"
done
