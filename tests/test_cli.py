"""The command-line surface (SPEC.md cli module): fit / render / eval / sweep, exit codes, config files.

CPU tests cover argument handling, usage and runtime error codes, config precedence and the PNG
conversions; the GPU tests run the commands end to end on tiny images."""
import csv
import os

import numpy as np
import pytest

from paper_2412_12734_b200 import cli


def _png(path, h=20, w=24, seed=0):
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w]
    img = np.stack([xx / (w - 1), yy / (h - 1), rng.random((h, w)) * 0.3], axis=2)
    cli.save_png(str(path), img)
    return str(path)


def test_png_round_trip_and_rounding(tmp_path):
    img = np.array([[[0.0, 0.5, 1.0], [-0.2, 1.7, 0.5 / 255.0]]])  # clamp, lround of x*255
    p = str(tmp_path / "a.png")
    cli.save_png(p, img)
    got = cli.load_png(p) * 255.0
    np.testing.assert_array_equal(np.rint(got), [[[0, 128, 255], [0, 255, 1]]])


def test_usage_errors_exit_2(tmp_path, capsys):
    assert cli.main(["fit", "--image", "x.png", "--sigma", "0"]) == 2
    assert cli.main(["fit", "--splats", "10"]) == 2  # no --image
    assert cli.main(["fit", "--image", "x.png", "--texture-res", "3"]) == 2  # N outside {1,2,4,8}
    assert cli.main(["render", "--splats", "s.gbil", "--out", "o.png", "--width", "8", "--height", "8",
                     "--background", "2,0,0"]) == 2
    assert cli.main(["nonsense"]) == 2
    cfg = tmp_path / "bad.cfg"
    cfg.write_text("no_such_key = 3\n")
    assert cli.main(["fit", "--image", "x.png", "--config", str(cfg)]) == 2
    assert "unknown key" in capsys.readouterr().err


def test_runtime_errors_exit_1(tmp_path, capsys):
    assert cli.main(["fit", "--image", str(tmp_path / "missing.png"), "--iters", "1"]) == 1
    assert "cannot open image" in capsys.readouterr().err
    junk = tmp_path / "junk.png"
    junk.write_bytes(b"not a png at all")
    assert cli.main(["eval", str(junk), str(junk)]) == 1
    assert "PNG" in capsys.readouterr().err


def test_config_file_precedence(tmp_path):
    cfg = tmp_path / "run.cfg"
    cfg.write_text("# comment\nsplats = 7\ntexture-res=2\nloss=mse-ssim\nforce-n = true\n")
    ap = cli._parser()
    a = cli._apply_config(ap, ["fit", "--image", "t.png", "--config", str(cfg)])
    assert (a.splats, a.texture_res, a.loss, a.force_n) == (7, 2, "mse-ssim", True)
    a = cli._apply_config(cli._parser(), ["fit", "--image", "t.png", "--config", str(cfg), "--splats", "9"])
    assert (a.splats, a.texture_res) == (9, 2)  # the command line wins


@pytest.mark.gpu
def test_fit_render_eval_end_to_end(tmp_path, capsys):
    img = _png(tmp_path / "t.png")
    out = tmp_path / "run"
    assert cli.main(["fit", "--image", img, "--splats", "40", "--iters", "25", "--texture-res", "2",
                     "--log-every", "5", "--out", str(out)]) == 0
    for f in ("splats.gbil", "metrics.csv", "render.png"):
        assert (out / f).exists(), f
    rows = list(csv.reader(open(out / "metrics.csv")))
    assert rows[0] == ["iter", "loss", "psnr", "ssim", "wall_ms"] and [int(r[0]) for r in rows[1:]] == [1, 5, 10, 15,
                                                                                                       20, 25]
    # the render of the written splats reproduces the fit's own final render byte for byte
    r = tmp_path / "r.png"
    assert cli.main(["render", "--splats", str(out / "splats.gbil"), "--out", str(r), "--width", "24",
                     "--height", "20"]) == 0
    assert r.read_bytes() == (out / "render.png").read_bytes()
    capsys.readouterr()
    assert cli.main(["eval", img, img]) == 0
    assert capsys.readouterr().out.strip() == "99.00,1.000000"
    # random colours are deterministic; the mip level renders the 1x1 downsampled grids
    r1, r2, r3 = (tmp_path / f"c{i}.png" for i in range(3))
    for p in (r1, r2):
        assert cli.main(["render", "--splats", str(out / "splats.gbil"), "--out", str(p), "--width", "24",
                         "--height", "20", "--random-colors", "42"]) == 0
    assert r1.read_bytes() == r2.read_bytes()
    assert cli.main(["render", "--splats", str(out / "splats.gbil"), "--out", str(r3), "--width", "24",
                     "--height", "20", "--mip-level", "1"]) == 0
    assert cli.main(["eval", str(r), str(r3)]) == 0
    psnr, ssim = (float(x) for x in capsys.readouterr().out.strip().split(","))
    assert psnr < 99.0  # the single-colour render differs


@pytest.mark.gpu
def test_sweep_degenerate_grid(tmp_path):
    img = _png(tmp_path / "t.png", seed=1)
    sw = tmp_path / "sw"
    assert cli.main(["sweep", "--image", img, "--splats", "30", "--iters", "15", "--sigmas", "0.5", "--ns", "2",
                     "--seeds", "2", "--out", str(sw)]) == 0
    rows = list(csv.reader(open(sw / "sweep.csv")))
    assert rows[0] == ["sigma", "n", "seed", "psnr", "ssim", "wall_seconds"] and len(rows) == 3
    summary = list(csv.reader(open(sw / "sweep_summary.csv")))
    assert summary[0] == ["sigma", "n", "median_psnr", "median_ssim"] and len(summary) == 2
    # one cell, seed 0: the same run as `fit` with that seed (up to the order of the gradient atomics)
    fit_dir = tmp_path / "fit"
    assert cli.main(["fit", "--image", img, "--splats", "30", "--iters", "15", "--texture-res", "2",
                     "--out", str(fit_dir)]) == 0
    last = list(csv.reader(open(fit_dir / "metrics.csv")))[-1]
    assert abs(float(rows[1][3]) - float(last[2])) < 0.05 and abs(float(rows[1][4]) - float(last[3])) < 1e-3
