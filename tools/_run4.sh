cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest4.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r2_pytest4.log | cut -c1-1500
