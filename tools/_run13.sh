cd $GRAFT_REPO_ROOT
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
for L in 4 6 3 8; do GB_LANES=$L $B > gpurun_out/r2_b13_l$L.json 2>>gpurun_out/r2_b13.err; python -c "
import json; d=json.loads(open('gpurun_out/r2_b13_l$L.json').read().strip().splitlines()[-1])
print('lanes $L', d['value'], d['ms_per_step'])"; done
