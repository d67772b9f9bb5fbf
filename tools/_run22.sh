cd $GRAFT_REPO_ROOT
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-cpp-host"
for r in a b; do
$B > gpurun_out/r2_b22_dl12_$r.json 2>>gpurun_out/r2_b22.err
for L in 8 16 20; do GB_LIB_PATH=variants/dl$L/libgb_raster.so $B > gpurun_out/r2_b22_dl${L}_$r.json 2>>gpurun_out/r2_b22.err; done
done
for f in gpurun_out/r2_b22_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], d['value'])"; done
