cd $GRAFT_REPO_ROOT
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_b9.json 2> gpurun_out/r2_b9.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2_b9.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e'], d['roofline']['frac'], d['cpu_baseline']['value'], d['clocks'])"
python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest9.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest9.log
