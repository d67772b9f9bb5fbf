"""The bounds-checked debug build (-DGB_DEBUG_CHECKS, libgb_raster_debug.so): every list entry must name a
primitive in [0, K) and every texel index must fall inside its n x n grid, else the kernel traps.  The
sanitizer case (tools/sanitize_case.py: binning, forward, loss, backward, Adam, SSIM/PSNR, GBIL, downsample
over both cameras and n in {1, 3, 8}) and the configs[3] trainer step run clean under it.  compute-sanitizer
is closed on the GPU pool, so this is the memory-safety check of the compositors."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2412_12734_b200", "libgb_raster_debug.so")


@pytest.mark.parametrize("script", ["tools/sanitize_case.py", "tools/debug_step.py"])
def test_debug_build_runs_clean(script):
    assert os.path.exists(LIB), "build the debug library (__graft_entry__.build())"
    env = dict(os.environ, GB_LIB_PATH=LIB)
    r = subprocess.run([sys.executable, os.path.join(ROOT, script)], env=env, capture_output=True, text=True,
                       timeout=900)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0
