"""Two configs[3]-size training steps (1M surfels, 8x8 textures, 8 views at 1600x1064; capacity binning,
CUDA graph, padded texel gradients, overlapped Adam) -- run under the bounds-checked debug build by
tests/test_gpu_debug_checks.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_12734_b200 as gb  # noqa: E402
import paper_2412_12734_b200.scenes as sc  # noqa: E402
from paper_2412_12734_b200.train import ViewShardedTrainer  # noqa: E402


def main():
    c = sc.baseline_config(3)
    s = gb.SplatSet.from_numpy(c.mode, gb.ColorGridConfig(c.n), **c.arrays())
    cams = [gb.PinholeCamera.from_spec(x) for x in c.cameras]
    views = list(range(8))
    tg = [torch.from_numpy(c.target(v)).cuda() for v in views]
    tr = ViewShardedTrainer(s, cams, views, graph=True)
    for _ in range(3):
        tr.step(tg)
    torch.cuda.synchronize()
    print("debug step ok", [round(float(x), 6) for x in tr.losses.cpu()][:3])


if __name__ == "__main__":
    main()
