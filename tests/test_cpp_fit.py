"""The training-loop half of the C++ drop-in (include/gbil_b200.hpp): gbil_b200::fit,
psnr/ssim and save/load_splats, against the reference's own fit (tests/golden/fit_cases.npz)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "fit_main.cpp")
LIBDIR = os.path.join(ROOT, "paper_2412_12734_b200")
GOLD = os.path.join(ROOT, "tests", "golden", "fit_cases.npz")
FIELDS = ("position", "depth_key", "theta", "log_scale", "opacity_logit", "grid")


def _build(tmp_path):
    exe = str(tmp_path / "fit_main")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe, "-L",
                    LIBDIR, "-lgb_raster", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def test_fit_dropin_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mse_n4", "ssim_n2"])
def test_cpp_fit_matches_reference_fit(tmp_path, name):
    d = np.load(GOLD)
    meta = d[f"{name}/meta"]
    W, H = int(meta[0]), int(meta[1])
    target = d[f"{name}/target"].astype(np.float64)
    inp = tmp_path / "in.bin"
    with open(inp, "wb") as fh:
        fh.write(np.asarray(meta, np.int64).tobytes())
        fh.write(target.tobytes())
    out = tmp_path / "out.bin"
    subprocess.run([_build(tmp_path), str(inp), str(out), str(tmp_path)], check=True)
    vals = []
    with open(out, "rb") as fh:
        for dt in [np.float64] * 8 + [np.int32]:
            n = int(np.frombuffer(fh.read(8), np.uint64)[0])
            vals.append(np.frombuffer(fh.read(n * np.dtype(dt).itemsize), dt))
    hist = vals[0].reshape(-1, 4)
    ref = d[f"{name}/history"]
    np.testing.assert_array_equal(hist[:, 0], ref[:, 0])
    np.testing.assert_allclose(hist[:, 1], ref[:, 1], rtol=1e-4)
    np.testing.assert_allclose(hist[:, 2], ref[:, 2], rtol=1e-5)
    np.testing.assert_allclose(hist[:, 3], ref[:, 3], rtol=1e-3, atol=1e-5)
    lr = {"position": 1.6e-4 * max(W, H), "theta": 1e-3, "log_scale": 5e-3, "opacity_logit": 5e-2,
          "grid": 2.5e-3, "depth_key": 1.0}
    for f, got in zip(FIELDS, vals[1:7]):
        r = d[f"{name}/final/{f}"].ravel()
        bad = np.abs(got - r) > 1e-5 * np.abs(r) + 0.02 * lr[f]
        assert bad.mean() <= 0.01, (f, int(bad.sum()))
    assert vals[8][0] == 1  # save -> load round trip exact
