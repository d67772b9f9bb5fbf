mkdir -p gpurun_out/ab
for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-cpp-host > gpurun_out/ab/new_$i.json 2> gpurun_out/ab/new_$i.err
  for v in pf1 pf3 pf5; do
    GB_LIB_PATH=variants/$v/libgb_raster.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-cpp-host > gpurun_out/ab/${v}_$i.json 2> gpurun_out/ab/${v}_$i.err
  done
done
