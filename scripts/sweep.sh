#!/bin/bash
# Executor-shape sweep on the GPU box: kernel_ms and roofline frac per
# SABLE_* setting.  usage: scripts/sweep.sh TAG CFG "ENV1;ENV2;..."
TAG=$1; CFG=$2; SETS=$3
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
IFS=';' read -ra ARR <<< "$SETS"
for S in "${ARR[@]}"; do
  echo "== $CFG $S" >> $OUT/sw.err; env $S timeout 600 python bench.py --config $CFG --steps 30 --warmup 5 --no-cpu-baseline > $OUT/sw.json 2>> $OUT/sw.err
  python -c "
import json,sys; d=json.load(open('$OUT/sw.json')); r=d['roofline']
print('$CFG', '$S'.ljust(70), 'kernel_ms=%.4f frac=%.3f items=%s tasks=%s chunks=%s bundles=%s fill=%s' % (r['kernel_ms'], r['frac'], d['config']['work_items'], d['config'].get('n_tasks'), d['config'].get('n_chunks'), d['config'].get('n_bundles'), d['config'].get('bundle_lane_fill')))
" 2>&1 | tail -1 | tee -a $OUT/sweep.txt
done
