cd $GRAFT_REPO_ROOT
python -m pytest tests/test_cpp_multiview.py -x -q > gpurun_out/r2_mv21.log 2>&1; echo "cpp mv rc=$?"; tail -3 gpurun_out/r2_mv21.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_b21.json 2> gpurun_out/r2_b21.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2_b21.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['cpp_host'])"
tail -3 gpurun_out/r2_b21.err
