#!/bin/bash
# Interleaved A/B of library variants on one box: bash tools/ab_run.sh ROUNDS name[=libpath] ...
# ("default" = the in-tree libgb_raster.so).  One bench line per (round, variant) in gpurun_out/ab_<name>_<r>.json.
R=$1; shift
rm -f gpurun_out/ab_*.json gpurun_out/ab_*.err
for r in $(seq 1 "$R"); do
  for v in "$@"; do
    name=${v%%=*}; lib=${v#*=}
    [ "$lib" = "$v" ] && lib=variants/$name/libgb_raster.so
    [ "$name" = default ] && lib=
    GB_LIB_PATH=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-cpp-host \
      > gpurun_out/ab_${name}_$r.json 2> gpurun_out/ab_${name}_$r.err
    python -c "import json,sys;d=json.loads(open('gpurun_out/ab_${name}_$r.json').read().strip().splitlines()[-1]);print('$name',$r,d['value'],d['roofline']['avg_launch_ms'])" || tail -3 gpurun_out/ab_${name}_$r.err
  done
done
