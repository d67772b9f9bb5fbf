#!/bin/bash
# Build an experimental variant of libgb_raster.so with extra nvcc flags into variants/<name>/
# (travels to the GPU box; select it with GB_LIB_PATH=variants/<name>/libgb_raster.so).  Delete variants
# after use: each is ~18 MB and the gpurun snapshot is capped at 512 MiB.
#   bash tools/build_variant.sh k4pf -DGB_K4_PREFETCH
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/variants/$NAME" "$ROOT/build/var_$NAME"
make -C "$ROOT/paper_2412_12734_b200/csrc" -j8 OUT="$ROOT/variants/$NAME/libgb_raster.so" MVHOST_OUT= \
  OBJDIR="$ROOT/build/var_$NAME" EXTRA="$*" 2>&1 | grep -E "error|spill.*k_backward_direct|spill.*k_forward_direct" || true
ls -la "$ROOT/variants/$NAME/libgb_raster.so"
