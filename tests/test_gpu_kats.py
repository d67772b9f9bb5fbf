"""The SPEC known-answer examples through the CUDA path, on one-splat ortho scenes.

Each KAT of the reference's texture and raster helpers (texture.hpp:27-111, raster.hpp:36-86;
SPEC.md:126-148, 204-236) is read off a rendered pixel: a single splat with theta = 0 and scales chosen so
that the pixel sees exactly the KAT's (u, v); with a black background the pixel's colour is alpha * c(u, v)
(alpha = alpha_k exp(-(u^2+v^2)/2) known in closed form), and a one-hot image gradient at that pixel turns
the backward into one adj_bilinear_accum call (texel gradients = c_hat * w, u_hat into the position
gradient).  Golden values: tests/golden/kat.json (produced by the compiled reference)."""
import json
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _one_splat(u, v, n, sigma, grid, alpha_k=0.8, W=64, H=64, no_thresholds=False):
    """A splat whose centre sits on the centre of pixel (32, 32); pixel (32 + dx, 32 + dy) sees (u, v)."""
    import paper_2412_12734_b200 as gb

    dx = 0 if u == 0 else int(math.copysign(12, u))
    dy = 0 if v == 0 else int(math.copysign(12, v))
    su = dx / u if u != 0 else 7.0
    sv = dy / v if v != 0 else 7.0
    arrays = dict(position=np.array([[32.5, 32.5]]), depth_key=np.zeros(1), theta=np.zeros(1),
                  log_scale=np.array([[math.log(su), math.log(sv)]]),
                  opacity_logit=np.array([math.log(alpha_k / (1 - alpha_k))]), grid=np.asarray(grid)[None, :])
    s = gb.SplatSet.from_numpy(gb.raster.MODE_ORTHO, gb.ColorGridConfig(n, sigma), **arrays)
    cam = gb.ImagePlaneCamera(W, H, (0.0, 0.0, 0.0))
    rc = gb.RasterConfig(16, 0.0, 0.0, 0.0, 1) if no_thresholds else gb.RasterConfig()
    b = gb.build_binning(s, cam, rc)
    out = gb.render_forward(s, cam, b)
    px, py = 32 + dx, 32 + dy
    # the fp32 scales the kernels use: u = dx / exp(float(log su))
    su32 = float(np.exp(np.float32(math.log(su)).astype(np.float64)))
    sv32 = float(np.exp(np.float32(math.log(sv)).astype(np.float64)))
    uu = dx / su32 if u != 0 else 0.0
    vv = dy / sv32 if v != 0 else 0.0
    a32 = float(1 / (1 + np.exp(-np.float64(np.float32(math.log(alpha_k / (1 - alpha_k)))))))
    alpha = min(a32 * math.exp(-0.5 * (uu * uu + vv * vv)), 0.999)
    return gb, s, cam, b, out, (px, py), alpha, (su32, sv32), (uu, vv)


def test_uv_to_grid_kats_through_cuda():  # SPEC.md:126-128, texture.hpp:27-47
    """A texture holding each texel's own (i_u, i_v) interpolates to the clamped grid coordinate
    (i_u + f_u, i_v + f_v): the pixel's colour / alpha reads uv_to_grid off the CUDA path."""
    kat = json.load(open(os.path.join(GOLD, "kat.json")))
    checked = 0
    for u, v, n, sigma, (iu, iv, fu, fv) in kat["uv_to_grid"]:
        if n < 2 or u * u + v * v > 40.0:  # n = 1 has no grid; G underflows fp32 beyond r^2 ~ 170 anyway
            continue
        grid = np.array([[i, j, 0.0] for i in range(n) for j in range(n)]).ravel()
        gb, s, cam, b, out, (px, py), alpha, _, _ = _one_splat(u, v, n, sigma, grid, no_thresholds=True)
        c = out.color[py, px].cpu().numpy().astype(np.float64) / alpha
        np.testing.assert_allclose(c[:2], [iu + fu, iv + fv], rtol=2e-5, atol=2e-5, err_msg=str((u, v, n, sigma)))
        checked += 1
    assert checked >= 4


def test_bilinear_kats_through_cuda():  # SPEC.md:136-138, texture.hpp:49-66
    kat = json.load(open(os.path.join(GOLD, "kat.json")))
    grid2 = np.array([0, 0, 0, 0, 0, 1, 1, 0, 0, 1, 0, 1], np.float64)  # C00, C01, C10, C11
    for u, v, want in kat["bilinear"]:
        gb, s, cam, b, out, (px, py), alpha, _, _ = _one_splat(u, v, 2, 0.5, grid2, no_thresholds=True)
        c = out.color[py, px].cpu().numpy().astype(np.float64) / alpha
        np.testing.assert_allclose(c, want, rtol=2e-5, atol=2e-6, err_msg=str((u, v)))
    # a constant grid renders its colour at any (u, v)
    gb, s, cam, b, out, (px, py), alpha, _, _ = _one_splat(0.17, -0.4, 4, 0.5, np.tile([0.3, 0.6, 0.9], 16))
    np.testing.assert_allclose(out.color[py, px].cpu().numpy() / alpha, [0.3, 0.6, 0.9], rtol=2e-6)


def test_adj_bilinear_kats_through_cuda():  # SPEC.md:146-148, texture.hpp:68-127, raster.hpp:338-360
    """One-hot image gradient g = c_hat / alpha at the pixel: K4's texel gradients are the KAT's c_hat * w
    and the position gradient is -(u_hat - alpha_hat alpha u) / s_u (theta = 0, raster.hpp:350-357)."""
    import torch

    from test_oracle_kat import bilinear

    kat = json.load(open(os.path.join(GOLD, "kat.json")))
    g8 = np.array(kat["adj_bilinear_grid8"])
    for u, v, c_hat, want_gg, want_uh, want_vh in kat["adj_bilinear"]:
        gb, s, cam, b, out, (px, py), alpha, (su, sv), (uu, vv) = _one_splat(u, v, 8, 0.5, g8)
        ig = torch.zeros((cam.height, cam.width, 3), device="cuda")
        ig[py, px] = torch.tensor(np.array(c_hat) / alpha, dtype=torch.float32)
        g = gb.render_backward(s, cam, b, out, ig)
        torch.cuda.synchronize()
        gg = g.grid.cpu().numpy().astype(np.float64).ravel()
        np.testing.assert_allclose(gg, want_gg, rtol=1e-5, atol=1e-6, err_msg=str((u, v)))
        col = bilinear(u, v, 8, 0.5, g8)
        alpha_hat = float(np.dot(np.array(c_hat) / alpha, col))  # T = 1, behind = black background
        uh = want_uh - alpha_hat * alpha * uu
        vh = want_vh - alpha_hat * alpha * vv
        pos = g.position.cpu().numpy().astype(np.float64).ravel()
        np.testing.assert_allclose(pos, [-uh / su, -vh / sv], rtol=1e-4, atol=1e-6, err_msg=str((u, v)))


def test_cull_kat_through_cuda():  # SPEC.md:224-226, raster.hpp:54-101
    """Pixel box [44,55] x [47,52] -> tiles (2..3) x (2..3); an off-screen and a sigmoid(-10) < 1/255 splat
    are culled (no tile lists them)."""
    import paper_2412_12734_b200 as gb

    arrays = dict(position=np.array([[50.0, 50.0], [-100.0, -100.0], [50.0, 50.0]]), depth_key=np.zeros(3),
                  theta=np.zeros(3), log_scale=np.array([[math.log(2.0), 0.0], [0.0, 0.0], [0.0, 0.0]]),
                  opacity_logit=np.array([0.0, 0.0, -10.0]), grid=np.zeros((3, 3)))
    s = gb.SplatSet.from_numpy(gb.raster.MODE_ORTHO, gb.ColorGridConfig(1), **arrays)
    b = gb.build_binning(s, gb.ImagePlaneCamera(100, 100), gb.RasterConfig())
    offsets, values = b.csr()
    tiles_x = 7
    listed = {t: values[offsets[t]:offsets[t + 1]].tolist() for t in range(len(offsets) - 1)
              if offsets[t + 1] > offsets[t]}
    assert listed == {ty * tiles_x + tx: [0] for ty in (2, 3) for tx in (2, 3)}


def test_forward_kats_through_cuda():  # SPEC.md:234-236, raster.hpp:237-254
    import paper_2412_12734_b200 as gb

    # two centred splats, the back one capped at alpha 0.999 (core.hpp:16): (0.5, 0.5 * 0.999, 0)
    arrays = dict(position=np.array([[8.5, 8.5], [8.5, 8.5]]), depth_key=np.array([0.0, 1.0]), theta=np.zeros(2),
                  log_scale=np.zeros((2, 2)), opacity_logit=np.array([0.0, 60.0]),
                  grid=np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]]))
    s = gb.SplatSet.from_numpy(gb.raster.MODE_ORTHO, gb.ColorGridConfig(1), **arrays)
    cam = gb.ImagePlaneCamera(16, 16)
    out = gb.render_forward(s, cam, gb.build_binning(s, cam, gb.RasterConfig(early_stop_transmittance=0.0)))
    np.testing.assert_allclose(out.color[8, 8].cpu().numpy(), [0.5, 0.5 * 0.999, 0.0], rtol=1e-6)
    assert int(out.last_rank[8, 8]) == 1
    # no splats: background everywhere, T = 1, last = -1
    empty = {k: v[:0] for k, v in arrays.items()}
    s0 = gb.SplatSet.from_numpy(gb.raster.MODE_ORTHO, gb.ColorGridConfig(1), **empty)
    cam0 = gb.ImagePlaneCamera(16, 16, (0.2, 0.4, 0.6))
    out0 = gb.render_forward(s0, cam0, gb.build_binning(s0, cam0, gb.RasterConfig()))
    np.testing.assert_allclose(out0.color.cpu().numpy(), np.broadcast_to([0.2, 0.4, 0.6], (16, 16, 3)), rtol=1e-7)
    assert bool((out0.final_transmittance == 1.0).all()) and bool((out0.last_rank == -1).all())


def test_adam_first_step_kat_through_cuda():  # SPEC.md:355-357, optim.hpp:84-88
    import paper_2412_12734_b200 as gb
    import torch

    a = json.load(open(os.path.join(GOLD, "kat.json")))["adam_first_step"]
    p = torch.tensor(a["p0"], dtype=torch.float32, device="cuda")
    g = torch.tensor(a["g"], dtype=torch.float32, device="cuda")
    m = torch.zeros(3, device="cuda")
    v = torch.zeros(3, device="cuda")
    flag = torch.full((1,), gb._lib.ADAM_FLAG_CLEAR, dtype=torch.int64, device="cuda")
    seg = (gb._lib.AdamSegment * 1)(gb._lib.AdamSegment(p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), 3, 4, 0))
    lrs = gb.LearningRates()
    lrs.color_grid = a["lr"]
    st = gb._lib.AdamStateC()
    st.t, st.beta1, st.beta2, st.epsilon = 0, 0.9, 0.999, 1e-8
    import ctypes as C

    ctx = gb.raster.context("cuda")
    for phase in (0, 1):
        gb._lib.check(gb._lib.lib.gb_adam_segments(ctx.handle, phase, seg, 1, C.byref(st), C.byref(lrs.to_c()),
                                                   flag.data_ptr()), "adam")
    torch.cuda.synchronize()
    np.testing.assert_allclose(p.cpu().numpy(), a["p1"], rtol=1e-6)
    np.testing.assert_allclose(m.cpu().numpy(), a["m"], rtol=1e-6)
    np.testing.assert_allclose(v.cpu().numpy(), a["v"], rtol=1e-5)
    assert st.t == 1
