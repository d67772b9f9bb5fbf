cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_strict.py -x -q -k "configs" > gpurun_out/r2_strict_big.log 2>&1; echo "strict rc=$?"
tail -8 gpurun_out/r2_strict_big.log | cut -c1-800
python -m pytest tests/test_gpu_configs4.py -x -q -k "4000000" > gpurun_out/r2_c4_big.log 2>&1; echo "c4 rc=$?"
tail -5 gpurun_out/r2_c4_big.log | cut -c1-1500
