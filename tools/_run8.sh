cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_train.py -x -q > gpurun_out/r2_t8.log 2>&1; echo "train rc=$?"; tail -3 gpurun_out/r2_t8.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
for r in a b; do
$B > gpurun_out/r2_b8_pad_$r.json 2>gpurun_out/r2_b8.err; echo "pad $r rc=$?"
GB_TEXEL_PAD=0 $B > gpurun_out/r2_b8_nopad_$r.json 2>>gpurun_out/r2_b8.err; echo "nopad $r rc=$?"
done
for f in pad_a nopad_a pad_b nopad_b; do python -c "
import json,sys; d=json.loads(open('gpurun_out/r2_b8_$f.json').read().strip().splitlines()[-1])
print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_ms'])"; done
ncu --set full --clock-control none --import-source on -k regex:"k_backward_direct" -c 1 -o gpurun_out/ncu_r02_pad_k4 -f python tools/ncu_pad_view.py > gpurun_out/ncu_pad.log 2>&1; echo "ncu rc=$?"
