"""The mip / random-colour diagnostics (texture.hpp:128-197, raster.hpp:394-400).

CPU: the output-size rules and their error messages, and the randomize_colors
stream, against the reference (compiled here) or its pinned values.  GPU: the
device downsample of seeded grids against the reference's downsample_grid
(tests/golden/diag_cases.npz), and render_random_colors end to end.
"""
import os
import re

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "diag_cases.npz")
SIZES = [(n, lv) for n in (1, 2, 3, 4, 5, 6, 8, 12, 16) for lv in range(0, 6)]


@pytest.mark.parametrize("n,levels", SIZES)
def test_downsample_size_rules(n, levels):
    import paper_2412_12734_b200.diagnostics as D

    if O.ref_available():
        ref = O.ref_downsample_grid(np.zeros(3 * n * n), n, levels)
        if isinstance(ref, str):
            with pytest.raises(ValueError, match=re.escape(ref)):
                D.downsample_size(n, levels)
        else:
            assert D.downsample_size(n, levels) == ref[1]
    else:  # pinned: halve while even, collapse an odd size to 1x1 when 2^(levels left) >= size
        cur, lv = n, levels
        while lv > 0 and cur > 1 and cur % 2 == 0:
            cur //= 2
            lv -= 1
        if lv > 0 and cur > 1:
            if (1 << lv) < cur:
                with pytest.raises(ValueError, match="not divisible by 2\\^levels"):
                    D.downsample_size(n, levels)
                return
            cur = 1
        assert D.downsample_size(n, levels) == cur


def test_negative_levels():
    import paper_2412_12734_b200.diagnostics as D

    with pytest.raises(ValueError, match="downsample_grid: negative level count"):
        D.downsample_size(4, -1)


def test_randomize_colors_stream():
    from paper_2412_12734_b200._lib import lib

    ours = np.zeros(7 * 27, np.float32)
    assert lib.gb_uniform_fill(5, ours.size, ours.ctypes.data) == 0
    ref = np.load(GOLD)["randomize/K7_n3_seed5"]
    np.testing.assert_array_equal(ours, ref.astype(np.float32))
    if O.ref_available():
        np.testing.assert_array_equal(ref, O.ref_randomize_colors(7, 3, 5))


@pytest.mark.gpu
def test_downsample_set_matches_reference():
    import torch

    import paper_2412_12734_b200 as gb
    import paper_2412_12734_b200.diagnostics as D

    d = np.load(GOLD)
    for key in sorted(k for k in d.files if k.endswith("/in")):
        name = key[:-3]
        n = int(round((d[key].shape[1] / 3) ** 0.5))
        levels = int(name.split("_l")[1])
        grids = d[key]
        K = grids.shape[0]
        s = gb.SplatSet(gb.raster.MODE_PINHOLE, gb.ColorGridConfig(n), position=torch.zeros(K, 3).cuda(),
                        quat=torch.zeros(K, 4).cuda(), log_scale=torch.zeros(K, 2).cuda(),
                        opacity_logit=torch.zeros(K).cuda(), grid=torch.as_tensor(grids).cuda())
        t = D.downsample_set(s, levels)
        assert t.grid_config.n == int(d[f"{name}/n_out"]), name
        # fp32 vs the reference's fp64 tree of 2x2 means: a few ulp
        np.testing.assert_allclose(t.grid.cpu().numpy(), d[f"{name}/out"], rtol=1e-6, atol=1e-7, err_msg=name)
        assert torch.equal(t.position, s.position)


@pytest.mark.gpu
def test_render_random_colors():
    import torch

    import paper_2412_12734_b200 as gb
    import paper_2412_12734_b200.diagnostics as D
    import paper_2412_12734_b200.scenes as sc

    arrays = sc.generate(O.MODE_ORTHO, 200, 4, 21, width=48, height=40, scale_lo=0.7, scale_hi=4.0)
    s = gb.SplatSet.from_numpy(O.MODE_ORTHO, gb.ColorGridConfig(4), **arrays)
    cam = gb.ImagePlaneCamera(48, 40)
    out = D.render_random_colors(s, cam, 77)
    r = D.randomize_colors(s, 77)
    ref = gb.render(r, cam)
    assert torch.equal(out.color, ref.color) and torch.equal(out.last_rank, ref.last_rank)
    assert not torch.equal(r.grid, s.grid) and torch.equal(r.theta, s.theta)
