cd $GRAFT_REPO_ROOT
python -c "import torch; print(torch.cuda.Stream.priority_range())"
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-cpp-host"
for r in a b; do
$B > gpurun_out/r2_b23_none_$r.json 2>>gpurun_out/r2_b23.err
GB_BIN_PRIORITY=-1 $B > gpurun_out/r2_b23_hi_$r.json 2>>gpurun_out/r2_b23.err
GB_BIN_PRIORITY=0 $B > gpurun_out/r2_b23_same_$r.json 2>>gpurun_out/r2_b23.err
done
for f in gpurun_out/r2_b23_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], d['value'])"; done
tail -3 gpurun_out/r2_b23.err
