cd $GRAFT_REPO_ROOT
python tools/diag_prim.py 4000000 1 > gpurun_out/diag_t1_fp32.json 2> gpurun_out/diag_t1_fp32.err; echo "diag rc=$?"
GB_LIB_PATH=paper_2412_12734_b200/libgb_raster_f64.so python tests/strict_case.py configs4_4000000_T1_rows8 gpurun_out/strict_configs4_4000000_T1_rows8.json > gpurun_out/r2_strict_t1.log 2>&1; echo "strict rc=$?"
tail -c 1200 gpurun_out/r2_strict_t1.log
cat gpurun_out/diag_t1_fp32.json | head -80
