cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_configs4.py -x -q > gpurun_out/r2_p16.log 2>&1; echo "c4 rc=$?"; tail -2 gpurun_out/r2_p16.log
python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2_p16b.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/r2_p16b.log
python -c "
import json
for f in ['parity_configs4_K4000000_T1','parity_configs4_K4000000_T16','parity_configs4_K1000000_T4','parity_configs2_fwd_bwd','parity_configs1_fwd_bwd']:
    d=json.load(open('gpurun_out/'+f+'.json')); print(f, d['image']['kink_pixels'], {k:(v['strict_violations_applicable'],v['model_violations'],v['kink_entries']) for k,v in d['grads'].items()})
"
