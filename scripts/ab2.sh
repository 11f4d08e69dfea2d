#!/bin/bash
# A/B over build variants and env knobs: scripts/ab2.sh TAG CFG "lib:ENV=..,ENV=.." ...
TAG=$1; CFG=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT; export SABLE_GEN_CACHE=/tmp/gencache
for v in "$@"; do
  lib=${v%%:*}; envs=${v#*:}; envs=${envs//,/ }
  [ "$lib" = "base" ] && lib=""
  name=${v//[:=, ]/_}
  env SABLE_LIB=$lib $envs timeout 400 python bench.py --config $CFG --steps 50 --warmup 5 --no-cpu-baseline > $OUT/b_${CFG}_${name}.json 2> $OUT/b_${CFG}_${name}.err
  python - <<PY
import json
try:
    d=json.load(open("$OUT/b_${CFG}_${name}.json"))
    print("$CFG", "$v", d["ms_per_step"], d["roofline"]["frac"], (d.get("l2_flushed") or {}).get("kernel_ms"))
except Exception as e:
    print("$CFG", "$v", "ERR", e)
PY
done
