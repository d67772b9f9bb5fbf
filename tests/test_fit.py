"""The image-fitting loop (train.hpp:22-219) and its metrics (metrics.hpp:167-191).

CPU: initialize() draws the reference's exact Rng sequence (bit-exact after the
fp32 rounding); TrainConfig validation messages.  GPU: SSIM (clamped and raw),
its gradient and PSNR against the reference's values; fit() against the
reference's own fit() on seeded targets (MSE and MSE + SSIM), through the logged
history and the final parameters; GBIL checkpoints.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "fit_cases.npz")
FIELDS = ("position", "depth_key", "theta", "log_scale", "opacity_logit", "grid")


@pytest.mark.skipif(not O.ref_available(), reason="compiled reference not present (GPU box)")
@pytest.mark.parametrize("w,h,K,n,seed", [(40, 32, 60, 4, 11), (7, 5, 50, 2, 3)])  # 50 > 35 px: warns
def test_initialize_matches_reference_draws(w, h, K, n, seed):
    import ctypes as C

    from paper_2412_12734_b200._lib import lib

    ref = O.ref_initialize(w, h, K, n, seed)
    ours = {f: np.zeros(v.shape, np.float32) for f, v in ref.items()}
    assert lib.gb_fit_initialize(w, h, K, n, seed, *[ours[f].ctypes.data for f in FIELDS]) == 0
    for f in FIELDS:
        np.testing.assert_array_equal(ours[f], ref[f].astype(np.float32), err_msg=f)
    assert len(np.unique(ours["depth_key"])) == K  # distinct keys (train.hpp:93-101)
    del C


def test_train_config_validation():
    import paper_2412_12734_b200.fit as F
    from paper_2412_12734_b200 import ColorGridConfig

    with pytest.raises(ValueError, match="splat_count must be >= 1"):
        F.TrainConfig(splat_count=0).validate()
    with pytest.raises(ValueError, match="one of 1, 2, 4, 8"):
        F.TrainConfig(grid=ColorGridConfig(3)).validate()
    F.TrainConfig(grid=ColorGridConfig(3), allow_any_n=True).validate()
    with pytest.raises(ValueError, match="log_every"):
        F.TrainConfig(log_every=0).validate()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["img_a", "img_b"])
def test_ssim_and_psnr_vs_reference(name):
    import torch

    import paper_2412_12734_b200.fit as F

    d = np.load(GOLD)
    a = torch.as_tensor(d[f"{name}/a"]).cuda()
    b = torch.as_tensor(d[f"{name}/b"]).cuda()
    assert abs(F.ssim(a, b) - float(d[f"{name}/ssim_clamped"])) <= 2e-6
    v, g = F.ssim_with_gradient(a, b)
    assert abs(v - float(d[f"{name}/ssim_raw"])) <= 2e-6
    ref_g = d[f"{name}/ssim_grad"]
    np.testing.assert_allclose(g.cpu().numpy(), ref_g, rtol=1e-3, atol=2e-4 * np.abs(ref_g).max())
    assert abs(F.psnr(a, b) - float(d[f"{name}/psnr"])) <= 1e-6 * float(d[f"{name}/psnr"])
    assert F.psnr(a, a) == 99.0  # metrics.hpp:176-178: identical images hit the cap
    assert abs(F.ssim(b, b) - 1.0) <= 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mse_n4", "ssim_n2", "mse_n1"])
def test_fit_matches_reference_fit(name):
    import torch

    import paper_2412_12734_b200.fit as F
    from paper_2412_12734_b200 import ColorGridConfig, RasterConfig

    d = np.load(GOLD)
    W, H, K, n, iters, ms, seed = [int(x) for x in d[f"{name}/meta"]]
    cfg = F.TrainConfig(splat_count=K, iterations=iters, seed=seed, grid=ColorGridConfig(n, 0.5), allow_any_n=True,
                        loss=F.LossKind.mse_plus_ssim if ms else F.LossKind.mse, log_every=1,
                        raster=RasterConfig(16))
    res = F.fit(torch.as_tensor(d[f"{name}/target"]).cuda(), cfg)
    hist = np.array([[r.iter, r.loss, r.psnr, r.ssim] for r in res.history])
    ref = d[f"{name}/history"]
    assert hist.shape == ref.shape
    np.testing.assert_array_equal(hist[:, 0], ref[:, 0])
    # fp32 rendering + fp32 loss sums vs the reference's fp64: ~1e-6 relative per iteration
    np.testing.assert_allclose(hist[:, 1], ref[:, 1], rtol=1e-4)
    np.testing.assert_allclose(hist[:, 2], ref[:, 2], rtol=1e-5)
    np.testing.assert_allclose(hist[:, 3], ref[:, 3], rtol=1e-3, atol=1e-5)
    # after `iters` Adam steps every parameter moved by <= iters*lr; the fp32 trajectory stays within a
    # small fraction of one step except where a near-zero gradient flips sign (Adam normalises it to a
    # full step), which must stay rare
    lr = {"position": 1.6e-4 * max(W, H), "theta": 1e-3, "log_scale": 5e-3, "opacity_logit": 5e-2,
          "grid": 2.5e-3, "depth_key": 1.0}
    got = {f: v.cpu().numpy().astype(np.float64) for f, v in res.splats.tensors().items()}
    for f in FIELDS:
        r = d[f"{name}/final/{f}"].reshape(got[f].shape)
        tol = 1e-5 * np.abs(r) + 0.02 * lr[f]
        bad = np.abs(got[f] - r) > tol
        assert bad.mean() <= 0.01, (f, int(bad.sum()), bad.size, float(np.abs(got[f] - r).max()))
    np.testing.assert_array_equal(got["depth_key"], d[f"{name}/final/depth_key"].astype(np.float32))


@pytest.mark.gpu
def test_fit_writes_gbil_checkpoints(tmp_path):
    import torch

    import paper_2412_12734_b200 as gb
    import paper_2412_12734_b200.fit as F

    d = np.load(GOLD)
    cfg = F.TrainConfig(splat_count=40, iterations=3, checkpoint_every=2, checkpoint_dir=str(tmp_path), log_every=2)
    res = F.fit(torch.as_tensor(d["mse_n4/target"]).cuda(), cfg)
    assert [r.iter for r in res.history] == [1, 2, 3]
    names = sorted(os.listdir(tmp_path))
    assert names == ["checkpoint_000002.gbil", "checkpoint_000002.history.csv", "checkpoint_000003.gbil",
                     "checkpoint_000003.history.csv"]
    last = gb.load_splats(str(tmp_path / "checkpoint_000003.gbil"))
    for f, v in res.splats.tensors().items():
        assert torch.equal(last.tensors()[f], v), f
    lines = open(tmp_path / "checkpoint_000003.history.csv").read().splitlines()
    assert lines[0] == "iter,loss,psnr" and len(lines) == 4
