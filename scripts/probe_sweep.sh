#!/bin/bash
# Dense-executor knob sweep on the calibration matrices (dense arm only).
# usage: scripts/probe_sweep.sh "h w fill lg" "ENV1;ENV2;..."
read -ra M <<< "$1"
IFS=';' read -ra ARR <<< "$2"
for S in "${ARR[@]}"; do
  echo "== $S"
  env PROBE_DELTAS=0 $S timeout 300 python scripts/calib_probe.py ${M[0]} ${M[1]} ${M[2]} ${M[3]} 2>&1 | tail -1
done
