"""SPEC known-answer tests on the oracle restatement (and the golden values
the compiled reference produced for the same inputs, tests/golden/kat.json)."""
import ctypes as C
import json
import math
import os

import numpy as np
import pytest

from parity import O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def uv_to_grid(u, v, n, s):
    iu, iv, fu, fv = C.c_int32(), C.c_int32(), C.c_double(), C.c_double()
    O.oracle_lib().orc_uv_to_grid(u, v, n, s, C.byref(iu), C.byref(iv), C.byref(fu), C.byref(fv))
    return iu.value, iv.value, fu.value, fv.value


def bilinear(u, v, n, s, grid):
    g = np.ascontiguousarray(grid, np.float64)
    c = np.zeros(3)
    O.oracle_lib().orc_bilinear(u, v, n, s, g.ctypes.data, c.ctypes.data)
    return c


def adj_bilinear(u, v, n, s, grid, c_hat):
    g = np.ascontiguousarray(grid, np.float64)
    ch = np.ascontiguousarray(c_hat, np.float64)
    gg = np.zeros_like(g)
    uh, vh = C.c_double(), C.c_double()
    O.oracle_lib().orc_adj_bilinear(u, v, n, s, g.ctypes.data, ch.ctypes.data, gg.ctypes.data, C.byref(uh),
                                    C.byref(vh))
    return gg, uh.value, vh.value


def test_uv_to_grid_spec_examples():
    assert uv_to_grid(-0.5, -0.5, 4, 0.5) == (0, 0, 0.0, 0.0)
    assert uv_to_grid(0.0, 0.0, 2, 0.5) == (0, 0, 0.5, 0.5)
    iu, iv, fu, fv = uv_to_grid(5.0, 0.0, 4, 0.5)
    assert (iu, fu) == (2, 1.0)


def test_bilinear_spec_examples():
    const = np.tile([0.3, 0.6, 0.9], 16)
    np.testing.assert_allclose(bilinear(0.17, -0.4, 4, 0.5, const), [0.3, 0.6, 0.9], rtol=1e-15)
    grid2 = np.array([0, 0, 0, 0, 0, 1, 1, 0, 0, 1, 0, 1], np.float64)  # C00, C01, C10, C11
    np.testing.assert_allclose(bilinear(0.0, 0.0, 2, 0.5, grid2), [0.5, 0.0, 0.5])
    np.testing.assert_allclose(bilinear(5.0, 0.0, 2, 0.5, grid2), [1.0, 0.0, 0.5])


def test_adj_bilinear_spec_examples():
    rng = np.random.default_rng(0)
    g = rng.random(4 * 4 * 3)
    _, uh, vh = adj_bilinear(0.9, 0.1, 4, 0.5, g, [1.0, 1.0, 1.0])  # |u| > sigma
    assert uh == 0.0
    _, uh, vh = adj_bilinear(0.1, 0.2, 4, 0.5, np.tile([0.2, 0.4, 0.6], 16), [1.0, -2.0, 0.5])
    assert uh == 0.0 and vh == 0.0
    # FD of sum(bilinear) wrt u, away from kinks
    for _ in range(50):
        u, v = rng.uniform(-0.45, 0.45, size=2)
        up = (4 - 1) * (u + 0.5) / 1.0
        if abs(up - round(up)) < 1e-2:
            continue
        _, uh, _ = adj_bilinear(u, v, 4, 0.5, g, [1.0, 1.0, 1.0])
        h = 1e-6
        fd = (bilinear(u + h, v, 4, 0.5, g).sum() - bilinear(u - h, v, 4, 0.5, g).sum()) / (2 * h)
        assert abs(uh - fd) <= 1e-4 * abs(fd) + 1e-6
    # partition of unity of the texel weights
    gg, _, _ = adj_bilinear(0.13, -0.21, 4, 0.5, g, [1.0, 2.0, 3.0])
    np.testing.assert_allclose(gg.reshape(-1, 3).sum(axis=0), [1.0, 2.0, 3.0], rtol=1e-14)


def test_intersect_ortho_spec_examples():
    u, v = C.c_double(), C.c_double()
    L = O.oracle_lib()
    L.orc_intersect_ortho(12.0, 20.0, 10.0, 20.0, 0.0, math.log(2.0), math.log(4.0), C.byref(u), C.byref(v))
    assert (u.value, v.value) == (1.0, 0.0)
    L.orc_intersect_ortho(10.0, 22.0, 10.0, 20.0, math.pi / 2, math.log(2.0), math.log(4.0), C.byref(u), C.byref(v))
    assert abs(u.value - 1.0) < 1e-15 and abs(v.value) < 1e-15
    L.orc_intersect_ortho(7.0, 3.0, 7.0, 3.0, 0.7, 0.3, -0.2, C.byref(u), C.byref(v))
    assert (u.value, v.value) == (0.0, 0.0)


def test_cull_spec_examples():
    arrays = dict(position=np.array([[50.0, 50.0], [-100.0, -100.0], [50.0, 50.0]]), depth_key=np.zeros(3),
                  theta=np.zeros(3), log_scale=np.array([[math.log(2.0), 0.0], [0.0, 0.0], [0.0, 0.0]]),
                  opacity_logit=np.array([0.0, 0.0, -10.0]), grid=np.zeros((3, 3)))
    scene = O.Scene64(arrays, 1)
    # box [44,56]x[47,53] -> pixel centres 44..55 x 47..52 (box_to_pixels, raster.hpp:93-101)
    depth, rect = O.project(scene, O.Cam(O.MODE_ORTHO, 100, 100), O.Cfg())
    assert rect[0].tolist() == [44, 55, 47, 52]
    assert rect[1].tolist() == [-1, -1, -1, -1]  # fully off-screen (on a 64x64 image in the SPEC)
    assert rect[2].tolist() == [-1, -1, -1, -1]  # sigmoid(-10) < 1/255


def test_gaussian_and_forward_examples():
    # single centred splat, constant grid c, alpha_k = 0.9 -> 0.9 c, T = 0.1
    c = np.array([0.3, 0.6, 0.9])
    arrays = dict(position=np.array([[8.5, 8.5]]), depth_key=np.zeros(1), theta=np.zeros(1),
                  log_scale=np.zeros((1, 2)), opacity_logit=np.array([math.log(9.0)]), grid=np.tile(c, 4)[None])
    scene = O.Scene64(arrays, 2)
    cam = O.Cam(O.MODE_ORTHO, 16, 16)
    cfg = O.Cfg()
    b = O.build_binning(scene, cam, cfg)
    f = O.render_forward(scene, cam, cfg, b)
    np.testing.assert_allclose(f["color"][8, 8], 0.9 * c, rtol=1e-14)
    assert abs(f["trans"][8, 8] - 0.1) < 1e-14
    # K = 0 -> background everywhere, T = 1
    empty = {k: v[:0] for k, v in arrays.items()}
    scene0 = O.Scene64(empty, 2)
    cam_bg = O.Cam(O.MODE_ORTHO, 16, 16, (0.2, 0.4, 0.6))
    b0 = O.build_binning(scene0, cam_bg, cfg)
    f0 = O.render_forward(scene0, cam_bg, cfg, b0)
    assert np.all(f0["color"] == np.array([0.2, 0.4, 0.6])) and np.all(f0["trans"] == 1.0)
    assert np.all(f0["last"] == -1)


def test_two_splat_composite_example():
    arrays = dict(position=np.array([[8.5, 8.5], [8.5, 8.5]]), depth_key=np.array([0.0, 1.0]), theta=np.zeros(2),
                  log_scale=np.zeros((2, 2)), opacity_logit=np.array([0.0, 60.0]),
                  grid=np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]]))
    scene = O.Scene64(arrays, 1)
    cam = O.Cam(O.MODE_ORTHO, 16, 16)
    cfg = O.Cfg(early_stop=0.0)
    b = O.build_binning(scene, cam, cfg)
    f = O.render_forward(scene, cam, cfg, b)
    # alpha_2 is capped at 0.999 (core.hpp:16), so green = 0.5*0.999
    np.testing.assert_allclose(f["color"][8, 8], [0.5, 0.5 * 0.999, 0.0], rtol=1e-12)


def test_zero_image_grad_gives_zero_gradients():
    import paper_2412_12734_b200.scenes as sc

    arrays = sc.generate(O.MODE_ORTHO, 40, 2, 3, width=32, height=32, scale_lo=1.0, scale_hi=5.0)
    scene = O.Scene64(arrays, 2)
    cam = O.Cam(O.MODE_ORTHO, 32, 32)
    cfg = O.Cfg()
    b = O.build_binning(scene, cam, cfg)
    f = O.render_forward(scene, cam, cfg, b)
    g, _, _ = O.render_backward(scene, cam, cfg, b, f, np.zeros((32, 32, 3)))
    for v in g.values():
        if v is not None:
            assert not v.any()


def test_adam_first_step_and_reference_golden():
    p, m, v, bad = O.adam_group(np.ones(4), np.ones(4), np.zeros(4), np.zeros(4), 0.1, 0.9, 0.999, 1e-8,
                                1 - 0.9, 1 - 0.999)
    np.testing.assert_allclose(p, 1.0 - 0.1, rtol=1e-6)
    assert bad == 0
    p, m, v, bad = O.adam_group(np.ones(3), np.array([0.0, np.nan, 1.0]), np.zeros(3), np.zeros(3), 0.1, 0.9,
                                0.999, 1e-8, 0.1, 0.001)
    assert bad == 2  # index 1 -> optim.hpp:81-83 throws naming the index
    kat = json.load(open(os.path.join(GOLD, "kat.json")))
    a = kat["adam_first_step"]
    p, m, v, _ = O.adam_group(np.array(a["p0"]), np.array(a["g"]), np.zeros(3), np.zeros(3), a["lr"], 0.9, 0.999,
                              1e-8, 1 - 0.9, 1 - 0.999)
    assert p.tolist() == a["p1"] and m.tolist() == a["m"] and v.tolist() == a["v"]


def test_texture_kats_match_reference_golden():
    kat = json.load(open(os.path.join(GOLD, "kat.json")))
    for u, v, n, s, exp in kat["uv_to_grid"]:
        assert list(uv_to_grid(u, v, n, s)) == exp
    grid2 = np.array([0, 0, 0, 0, 0, 1, 1, 0, 0, 1, 0, 1], np.float64)
    for u, v, exp in kat["bilinear"]:
        assert bilinear(u, v, 2, 0.5, grid2).tolist() == exp
    g8 = np.array(kat["adj_bilinear_grid8"])
    for u, v, ch, gg, uh, vh in kat["adj_bilinear"]:
        ggo, uho, vho = adj_bilinear(u, v, 8, 0.5, g8, ch)
        assert ggo.tolist() == gg and uho == uh and vho == vh


def test_l1_loss():
    c = np.array([0.5, 0.2, 0.9, 0.4]); t = np.array([0.1, 0.2, 1.0, 0.3])
    val, grad = O.l1_loss(c, t, 0.25)
    assert abs(val - 0.25 * (0.4 + 0.0 + 0.1 + 0.1)) < 1e-15
    assert grad.tolist() == [0.25, 0.0, -0.25, 0.25]
