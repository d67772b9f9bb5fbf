cd $GRAFT_REPO_ROOT
free -g | head -2; nproc
python -m pytest tests/test_gpu_strict.py -x -q -k "ortho_n3 or pinhole_small" > gpurun_out/r2_strict_small.log 2>&1; echo "strict rc=$?"
tail -30 gpurun_out/r2_strict_small.log | cut -c1-600
python -m pytest tests/test_gpu_configs4.py -x -q -k "1000000" > gpurun_out/r2_c4_small.log 2>&1; echo "c4 rc=$?"
tail -5 gpurun_out/r2_c4_small.log | cut -c1-1500
