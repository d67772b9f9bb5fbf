"""The C++ drop-in header (include/gbil_b200.hpp): compiles against the C-ABI
here, and on a GPU reproduces the reference API end to end (bit-exact tile
lists, image and gradients within tolerance of the fp64 oracle, and the
reference's std::invalid_argument on a size mismatch)."""
import os
import subprocess

import numpy as np
import pytest

from parity import O, compare_grads, compare_image

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_main.cpp")
LIBDIR = os.path.join(ROOT, "paper_2412_12734_b200")


def _build(tmp_path):
    exe = str(tmp_path / "dropin_main")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe, "-L", LIBDIR,
                    "-lgb_raster", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def test_dropin_header_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


def _read(path):
    dts = [np.float32] * 6 + [np.int64, np.int32] + [np.float64, np.float64, np.int32, np.float64] + \
          [np.float64] * 5 + [np.int32]
    out = []
    with open(path, "rb") as fh:
        for dt in dts:
            n = int(np.frombuffer(fh.read(8), np.uint64)[0])
            out.append(np.frombuffer(fh.read(n * np.dtype(dt).itemsize), dt))
    return out


@pytest.mark.gpu
def test_dropin_matches_oracle(tmp_path):
    exe = _build(tmp_path)
    res = str(tmp_path / "out.bin")
    subprocess.run([exe, res], check=True)
    pos, dk, th, ls, op, gr, offs, vals, color, trans, last, ig, gp, gt, gl, go, gg, threw = _read(res)
    K, n, W, H = 2000, 4, 160, 120
    arrays = dict(position=pos.reshape(K, 2), depth_key=dk, theta=th, log_scale=ls.reshape(K, 2),
                  opacity_logit=op, grid=gr.reshape(K, -1))
    cam = O.Cam(O.MODE_ORTHO, W, H, (0.1, 0.2, 0.3))
    cfg = O.Cfg()
    scene = O.Scene64(arrays, n)
    b = O.build_binning(scene, cam, cfg)
    assert np.array_equal(b[0], offs) and np.array_equal(b[1], vals)
    f = O.render_forward(scene, cam, cfg, b)
    gpu = dict(color=color.reshape(H, W, 3), trans=trans.reshape(H, W), last=last.reshape(H, W))
    im = compare_image(gpu, dict(color=f["color"], trans=f["trans"], last=f["last"], kink=f["kink"]))
    assert im["color_violations"] == 0 and im["last_rank_mismatch"] == 0, im
    g, mag, slack = O.render_backward(scene, cam, cfg, b, f, ig.reshape(H, W, 3))
    st = compare_grads(dict(grads=dict(position=gp, theta=gt, log_scale=gl, opacity_logit=go, grid=gg)),
                       dict(grads=g, mag=mag, slack=slack))
    for k, v in st.items():
        assert v["strict_violations_applicable"] == 0 and v["model_violations"] == 0, (k, v)
    assert threw[0] == 1
