"""Print the K4 development counters for one configs[3] view (needs variants/dbg/libgb_raster.so from
tools/dbg_counters.sh, or GB_LIB_PATH pointing at another -DGB_DEBUG_COUNTERS build)."""
import ctypes as C, os, sys
os.environ.setdefault("GB_LIB_PATH", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "variants",
                                                 "dbg", "libgb_raster.so"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2412_12734_b200 as gb, paper_2412_12734_b200.scenes as sc
from paper_2412_12734_b200 import _lib
c = sc.baseline_config(3)
splats = gb.SplatSet.from_numpy(c.mode, gb.ColorGridConfig(c.n), **c.arrays())
cam = gb.PinholeCamera.from_spec(c.cameras[0])
b = gb.build_binning(splats, cam, gb.RasterConfig())
out = gb.render_forward(splats, cam, b)
loss, ig = gb.l1_loss(out.color, torch.as_tensor(c.target(0)).cuda())
cnt = (C.c_ulonglong * 8)()
_lib.lib.gb_debug_counters(cnt, 1)
g = gb.render_backward(splats, cam, b, out, ig)
torch.cuda.synchronize()
_lib.lib.gb_debug_counters(cnt, 0)
v = list(cnt)
print("P", b.total, "warp-entries", v[0], "box-pass", v[1], "active", v[2], "active lanes", v[3],
      "uniform groups", v[4], "per-lane groups", v[5], "lanes/active", v[3] / max(1, v[2]),
      "both 4x4 halves", v[6] / max(1, v[2]), "both 8x2 halves", v[7] / max(1, v[2]))
