#!/bin/bash
# builds a counter-instrumented copy of libgb_raster.so into build/dbg and prints the K4 counters for one view
set -e
cd "$(dirname "$0")/.."
mkdir -p build/dbg tools/_dbg
for f in gb_capi gb_project gb_binning gb_misc gb_composite gb_metrics gb_texture gb_io; do cp build/obj/$f.o build/dbg/; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DGB_DEBUG_COUNTERS -c paper_2412_12734_b200/csrc/gb_raster.cu -o build/dbg/gb_raster.o
g++ -std=c++17 -O2 -fPIC -c paper_2412_12734_b200/csrc/gb_scene.cpp -o build/dbg/gb_scene.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/_dbg/libgb_raster.so build/dbg/*.o
