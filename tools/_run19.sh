cd $GRAFT_REPO_ROOT
python tools/parity_sweep4.py > gpurun_out/sweep4_fp32.log 2>&1; echo "fp32 sweep rc=$?"; cat gpurun_out/sweep4_fp32.log | grep -E "OK|FAIL" | cut -c1-200
GB_LIB_PATH=paper_2412_12734_b200/libgb_raster_f64.so python tools/parity_sweep4.py --strict > gpurun_out/sweep4_strict.log 2>&1; echo "strict sweep rc=$?"; grep -E "OK|FAIL" gpurun_out/sweep4_strict.log | cut -c1-200
