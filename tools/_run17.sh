cd $GRAFT_REPO_ROOT
timeout 1500 python tools/diag_pixels.py 4000000 1 2626617 > gpurun_out/diag_pixels.json 2> gpurun_out/diag_pixels.err; echo "diag rc=$?"
head -c 4000 gpurun_out/diag_pixels.json; tail -3 gpurun_out/diag_pixels.err
python -m pytest tests/test_gpu_debug_checks.py -x -q > gpurun_out/r2_dbg17.log 2>&1; echo "debug rc=$?"; tail -3 gpurun_out/r2_dbg17.log
