"""Distribution of tile-list lengths (pairs per tile) of one view of a configs[4] cell.
    python tools/bucket_hist.py [count] [n]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2412_12734_b200 as gb  # noqa: E402
import paper_2412_12734_b200.scenes as sc  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
c = sc.baseline_config(4, count=count, n=n)
s = gb.SplatSet.from_numpy(c.mode, gb.ColorGridConfig(c.n), **c.arrays())
cam = gb.PinholeCamera.from_spec(c.cameras[0])
b = gb.build_binning(s, cam, gb.RasterConfig())
off, _ = b.csr()
L = np.diff(off)
q = np.percentile(L, [50, 90, 99, 99.9, 100])
print(f"K={count} tiles={len(L)} pairs={L.sum()} mean={L.mean():.0f} p50/p90/p99/p99.9/max={q.round().tolist()}")
for t in (128, 512, 2048, 8192, 32768):
    m = L > t
    print(f"  > {t}: {m.sum()} tiles, {L[m].sum() / max(1, L.sum()):.3f} of the pairs")
