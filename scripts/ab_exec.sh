#!/bin/bash
# A/B of the SpMV executors on the GPU box: bench lines per config and executor.
# usage: scripts/ab_exec.sh TAG "c2 c4" "unit staged" [extra env per run]
TAG=$1; CFGS=$2; EXECS=$3
OUT=gpurun_out/$TAG; mkdir -p $OUT
export SABLE_GEN_CACHE=/tmp/gencache
for c in $CFGS; do for ex in $EXECS; do
  name=${ex//[:= ]/_}
  envs=${ex//:/ }
  env SABLE_EXEC=${envs} timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline \
    > $OUT/b_${c}_${name}.json 2> $OUT/b_${c}_${name}.err
  echo "$c $ex rc=$? $(python -c "import json,sys; d=json.load(open('$OUT/b_${c}_${name}.json')); print(d['ms_per_step'], d['roofline']['frac'])" 2>/dev/null)"
done; done
