mkdir -p gpurun_out/$1; export SABLE_GEN_CACHE=/tmp/gencache
shift_name=$1; shift
for c in $CONFIGS; do for v in "$@"; do
  lib=${v%%:*}; envs=${v#*:}
  [ "$lib" = "base" ] && lib=""
  env SABLE_LIB=$lib $envs timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/$shift_name/b_${c}_${v//[:= ]/_}.json 2> gpurun_out/$shift_name/b_${c}_${v//[:= ]/_}.err
done; done
