cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_configs4.py -x -q -k "4000000-1" > gpurun_out/r2_c4_t1b.log 2>&1; echo "c4 t1 rc=$?"; tail -3 gpurun_out/r2_c4_t1b.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$B > gpurun_out/r2_b6_direct_a.json 2>gpurun_out/r2_b6_direct_a.err; echo "direct a rc=$?"
GB_LIB_PATH=variants/stage/libgb_raster.so $B > gpurun_out/r2_b6_stage_a.json 2>gpurun_out/r2_b6_stage_a.err; echo "stage a rc=$?"
$B > gpurun_out/r2_b6_direct_b.json 2>>gpurun_out/r2_b6_direct_a.err; echo "direct b rc=$?"
GB_LIB_PATH=variants/stage/libgb_raster.so $B > gpurun_out/r2_b6_stage_b.json 2>>gpurun_out/r2_b6_stage_a.err; echo "stage b rc=$?"
for f in direct_a stage_a direct_b stage_b; do python -c "
import json,sys; d=json.loads(open('gpurun_out/r2_b6_$f.json').read().strip().splitlines()[-1])
print('$f', d['value'], d['ms_per_step'], d['e2e']['value'] if d.get('e2e') else None, d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['kernel_ms_per_step'], d.get('collective_ms'))"; done
ncu --set full --clock-control none --import-source on -k regex:"k_backward_direct|k_forward_direct" -c 2 -o gpurun_out/ncu_r02_stage_k34 -f env GB_LIB_PATH=variants/stage/libgb_raster.so python tools/ncu_view.py > gpurun_out/ncu_stage.log 2>&1; echo "ncu stage rc=$?"
ncu --set full --clock-control none --import-source on -o gpurun_out/ncu_r02_all -f python tools/ncu_view.py > gpurun_out/ncu_all.log 2>&1; echo "ncu all rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
ls -la gpurun_out/*.ncu-rep
