cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_configs4.py tests/test_gpu_parity.py tests/test_gpu_strict.py -q > gpurun_out/r2_p18.log 2>&1; echo "parity rc=$?"; tail -4 gpurun_out/r2_p18.log
python -c "
import json
for f in ['parity_configs4_K4000000_T1','parity_configs4_K4000000_T16','parity_configs4_K1000000_T4','parity_configs2_fwd_bwd','parity_configs1_fwd_bwd','strict_configs2','strict_configs4_1000000_T16_rows8']:
    try:
        d=json.load(open('gpurun_out/'+f+'.json')); print(f, d['image']['kink_pixels'], {k:(v['strict_violations'],v['strict_violations_applicable'],v['model_violations'],v['kink_entries']) for k,v in d['grads'].items()})
    except Exception as e: print(f, e)
"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
