cd $GRAFT_REPO_ROOT
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-graph > gpurun_out/r2_b11_nograph.json 2>gpurun_out/r2_b11.err; echo "nograph rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2_b11_nograph.json').read().strip().splitlines()[-1])
print('nograph', d['value'], d['ms_per_step'], d['e2e'])"
