cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_strict.py -x -q -k "ortho_n3 or pinhole_small" > gpurun_out/r2_s10.log 2>&1; echo "strict rc=$?"; tail -2 gpurun_out/r2_s10.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$B > gpurun_out/r2_b10_eager.json 2>gpurun_out/r2_b10.err; echo "eager rc=$?"
GB_GRAPH_HOST=1 $B > gpurun_out/r2_b10_ghost.json 2>>gpurun_out/r2_b10.err; echo "ghost rc=$?"
for f in eager ghost; do python -c "
import json; d=json.loads(open('gpurun_out/r2_b10_$f.json').read().strip().splitlines()[-1])
print('$f', d['value'], d['ms_per_step'], d['e2e'])"; done
