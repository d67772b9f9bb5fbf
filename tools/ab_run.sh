#!/bin/bash
# Interleaved A/B on one box: bash tools/ab_run.sh ROUNDS spec ...
#   spec = name              -> variants/<name>/libgb_raster.so ("default" = the in-tree library)
#        = name=path         -> that library
#        = name:VAR=val[,VAR=val] -> the in-tree library with trainer/bench environment switches
# One bench line per (round, spec) in gpurun_out/ab_<name>_<r>.json.
R=$1; shift
rm -f gpurun_out/ab_*.json gpurun_out/ab_*.err
for r in $(seq 1 "$R"); do
  for v in "$@"; do
    envs=
    case $v in
      *:*) name=${v%%:*}; envs=${v#*:}; lib= ;;
      *=*) name=${v%%=*}; lib=${v#*=} ;;
      default) name=default; lib= ;;
      *) name=$v; lib=variants/$v/libgb_raster.so ;;
    esac
    env GB_LIB_PATH=$lib ${envs//,/ } timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
      --no-cpp-host > gpurun_out/ab_${name}_$r.json 2> gpurun_out/ab_${name}_$r.err
    python -c "import json,sys;d=json.loads(open('gpurun_out/ab_${name}_$r.json').read().strip().splitlines()[-1]);print('$name',$r,d['value'],d['roofline']['avg_launch_ms'])" || tail -3 gpurun_out/ab_${name}_$r.err
  done
done
