cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_configs4.py -x -q -k "4000000-1" > gpurun_out/r2_c4_t1.log 2>&1; echo "c4 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/parity_configs4_K4000000_T1.json'))
for f,v in d['grads'].items(): print(f, v['strict_violations_applicable'], v['model_violations'], v['applicable'], v['model_list'])
"
GB_LIB_PATH=paper_2412_12734_b200/libgb_raster_f64.so python tests/strict_case.py configs4_4000000_T1_rows8 gpurun_out/strict_configs4_4000000_T1_rows8.json > gpurun_out/r2_strict_t1.log 2>&1; echo "strict rc=$?"
tail -c 1500 gpurun_out/r2_strict_t1.log
