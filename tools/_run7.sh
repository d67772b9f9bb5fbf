cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py tests/test_gpu_kats.py -x -q > gpurun_out/r2_p7.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/r2_p7.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
for r in a b; do
$B > gpurun_out/r2_b7_ws_$r.json 2>gpurun_out/r2_b7.err; echo "ws $r rc=$?"
GB_LIB_PATH=variants/nows/libgb_raster.so $B > gpurun_out/r2_b7_nows_$r.json 2>>gpurun_out/r2_b7.err; echo "nows $r rc=$?"
done
for f in ws_a nows_a ws_b nows_b; do python -c "
import json,sys; d=json.loads(open('gpurun_out/r2_b7_$f.json').read().strip().splitlines()[-1])
print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_ms'])"; done
ncu --set full --clock-control none --import-source on -k regex:"k_backward_direct|k_forward_direct" -c 2 -o gpurun_out/ncu_r02_ws_k34 -f python tools/ncu_view.py > gpurun_out/ncu_ws.log 2>&1; echo "ncu rc=$?"
