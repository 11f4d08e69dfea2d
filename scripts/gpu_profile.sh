#!/bin/bash
# Run on the GPU box (via gpurun): GPU tests, bench lines per config, the ncu
# launch list and one full ncu capture of the SpMV kernel per config.
# usage: scripts/gpu_profile.sh TAG "c2 c4" [tests]
set -u
TAG=${1:-r02}
CFGS=${2:-"c2"}
TESTS=${3:-tests}
NCU=${4:-ncu}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
if [ "$TESTS" = tests ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $OUT/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/gpu_tests.log
fi
for c in $CFGS; do
  timeout 900 python bench.py --config $c --steps 50 --warmup 5 > $OUT/bench_$c.json 2> $OUT/bench_$c.err; rc=$?
  echo "bench $c rc=$rc"; tail -c 1500 $OUT/bench_$c.json
  if [ $rc -eq 0 ] && [ "$NCU" = ncu ]; then
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $OUT/launches_$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline \
      > $OUT/ncu_launch_$c.log 2>&1; echo "ncu launches $c rc=$?"
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:unit_kernel -s 3 -c 1 \
      -o $OUT/unit_$c python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline \
      > $OUT/ncu_full_$c.log 2>&1; echo "ncu full $c rc=$?"
  fi
done
ls -la $OUT
