#!/bin/bash
# Development aid: a copy of libgb_raster.so with IEEE reciprocal/exp2 in the shared evaluation
# (GB_PRECISE_EVAL) into tools/_precise/, for A/B numerics runs (GB_LIB_PATH=tools/_precise/libgb_raster.so).
set -e
cd "$(dirname "$0")/.."
mkdir -p build/precise tools/_precise
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -DGB_PRECISE_EVAL"
for f in gb_capi gb_binning gb_raster gb_composite gb_misc gb_metrics gb_texture gb_io; do
  nvcc $F -c paper_2412_12734_b200/csrc/$f.cu -o build/precise/$f.o &
done
nvcc $F -fmad=false -c paper_2412_12734_b200/csrc/gb_project.cu -o build/precise/gb_project.o &
g++ -std=c++17 -O2 -fPIC -fvisibility=hidden -ffp-contract=off -c paper_2412_12734_b200/csrc/gb_scene.cpp -o build/precise/gb_scene.o &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/_precise/libgb_raster.so build/precise/*.o -Xlinker --exclude-libs,ALL
