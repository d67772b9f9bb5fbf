"""A small end-to-end case for compute-sanitizer (memcheck / racecheck / synccheck), one tool per run:
binning, forward, L1, backward, Adam, SSIM/PSNR, GBIL save/load, downsample.

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_case.py
"""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2412_12734_b200 as gb
import paper_2412_12734_b200.diagnostics as D
import paper_2412_12734_b200.fit as F
import paper_2412_12734_b200.scenes as sc


def run(mode, n):
    if mode == gb.raster.MODE_PINHOLE:
        arrays = sc.generate(mode, 1500, n, 3, scale_lo=0.02, scale_hi=0.15)
        cam = gb.PinholeCamera.from_spec(sc.look_at((0.3, -0.2, -3.0), (0, 0, 0), 90, 70, 80.0, 80.0, 45.0, 35.0))
    else:
        arrays = sc.generate(mode, 1500, n, 4, width=90, height=70, scale_lo=0.5, scale_hi=5.0)
        cam = gb.ImagePlaneCamera(90, 70, (0.1, 0.2, 0.3))
    s = gb.SplatSet.from_numpy(mode, gb.ColorGridConfig(n), **arrays)
    b = gb.build_binning(s, cam)
    out = gb.render_forward(s, cam, b)
    target = torch.rand((70, 90, 3), device="cuda")
    loss, ig = gb.l1_loss(out.color, target)
    g = gb.render_backward(s, cam, b, out, ig)
    gb.adam_step(s, g, gb.AdamState(s), gb.LearningRates())
    torch.cuda.synchronize()
    return s, out, target


def main():
    for mode in (gb.raster.MODE_PINHOLE, gb.raster.MODE_ORTHO):
        for n in (1, 3, 8):
            s, out, target = run(mode, n)
    F.ssim_with_gradient(out.color, target)
    F.psnr(out.color, target)
    D.downsample_set(s, 2)
    with tempfile.TemporaryDirectory() as d:
        gb.save_splats(os.path.join(d, "a.gbil"), s)
        gb.load_splats(os.path.join(d, "a.gbil"))
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
