#!/bin/bash
# Builds the counter-instrumented K4 (-DGB_DEBUG_COUNTERS) into variants/dbg/ and prints the counters for one
# configs[3] view on the GPU:  bash tools/dbg_counters.sh && GB_LIB_PATH=variants/dbg/libgb_raster.so python tools/dbg_run.py
set -e
cd "$(dirname "$0")/.."
bash tools/build_variant.sh dbg -DGB_DEBUG_COUNTERS
