cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/r2_b14.json 2> gpurun_out/r2_b14.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2_b14.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e'], d['roofline']['frac'], d['cpu_baseline'], d['clocks'])"
python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest14.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest14.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke14.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_smoke14.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_r02_final.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch14.log 2>&1; echo "ncu launch rc=$?"
ncu --set full --clock-control none --import-source on -o gpurun_out/ncu_r02_final_all -f python tools/ncu_pad_view.py > gpurun_out/ncu_final_all.log 2>&1; echo "ncu all rc=$?"
grep "ncu_view ok" gpurun_out/ncu_final_all.log
