"""The C++ view-sharded training step (include/gbil_b200.hpp, gbil_b200::multiview): one host thread per
GPU, NCCL communicators through the C-ABI (gb_comm_init_all), reduce-scatter -> Adam on the rank's slice
-> all-gather, or all-reduce -> Adam.  On one B200 (ncclCommInitAll over one device) its gradients, losses
and parameters match the Python trainer's (ViewShardedTrainer) on the same inputs."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "multiview_main.cpp")
LIBDIR = os.path.join(ROOT, "paper_2412_12734_b200")
GROUPS = ("position", "quat", "log_scale", "opacity_logit", "grid")


def _build(tmp_path):
    exe = str(tmp_path / "multiview_main")
    subprocess.run(["g++", "-std=c++20", "-O2", "-pthread", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
                    "-L", LIBDIR, "-lgb_raster", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def test_multiview_host_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


def _inputs(path):
    import paper_2412_12734_b200.scenes as sc

    K, n, W, H, V = 20_000, 4, 192, 128, 4
    arrays = sc.generate(sc.MODE_PINHOLE, K, n, 3, mean_sigma=1.0, scale_lo=0.005, scale_hi=0.05)
    cams = sc.fibonacci_cameras(V, 4.0, W, H, 160.0, 160.0, W / 2, H / 2)
    targets = [sc.uniform_image(40 + v, W, H) for v in range(V)]
    with open(path, "wb") as fh:
        fh.write(np.int64(K).tobytes())
        fh.write(np.array([n, W, H, V], np.int32).tobytes())
        for f in GROUPS:
            fh.write(np.ascontiguousarray(arrays[f], np.float32).tobytes())
        for c in cams:
            fh.write(np.array([c.fx, c.fy, c.cx, c.cy, *np.asarray(c.rot).ravel(), *np.asarray(c.trans)],
                              np.float64).tobytes())
        for t in targets:
            fh.write(np.ascontiguousarray(t, np.float32).tobytes())
    return K, n, arrays, cams, targets


def _outputs(path, steps):
    raw = open(path, "rb").read()
    losses = np.frombuffer(raw[:8 * steps], np.float64)
    T = int(np.frombuffer(raw[8 * steps:8 * steps + 8], np.int64)[0])
    o = 8 * steps + 8
    params = np.frombuffer(raw[o:o + 4 * T], np.float32)
    grads = np.frombuffer(raw[o + 4 * T:o + 8 * T], np.float32)
    offs = np.frombuffer(raw[o + 8 * T:o + 8 * T + 40], np.int64)
    return losses, params, grads, dict(zip(GROUPS, offs))


@pytest.mark.gpu
@pytest.mark.parametrize("sharded,steps", [(False, 1), (True, 2)])
def test_multiview_cpp_matches_python_trainer(tmp_path, sharded, steps):
    import torch

    import paper_2412_12734_b200 as gb
    from paper_2412_12734_b200.train import ViewShardedTrainer

    exe = _build(tmp_path)
    K, n, arrays, cams, targets = _inputs(str(tmp_path / "in.bin"))
    r = subprocess.run([exe, str(tmp_path / "in.bin"), str(tmp_path / "out.bin"), str(steps), str(int(sharded)), "0"],
                       capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0
    losses, params, grads, offs = _outputs(str(tmp_path / "out.bin"), steps)

    s = gb.SplatSet.from_numpy(gb.raster.MODE_PINHOLE, gb.ColorGridConfig(n), **arrays)
    lrs = gb.LearningRates()
    lrs.position *= 6.0
    tr = ViewShardedTrainer(s, [gb.PinholeCamera.from_spec(c) for c in cams], list(range(len(cams))), lrs=lrs,
                            async_binning=False, lanes=1, sharded_adam=sharded, overlap_adam=False)
    tg = [torch.as_tensor(t).cuda() for t in targets]
    want_losses = []
    for _ in range(steps):
        want_losses.append(float(tr.step(tg).sum()))
    torch.cuda.synchronize()
    np.testing.assert_allclose(losses, want_losses, rtol=1e-5)
    sizes = dict(position=3 * K, quat=4 * K, log_scale=2 * K, opacity_logit=K, grid=K * 3 * n * n)
    for f in GROUPS:
        got_p = params[offs[f]:offs[f] + sizes[f]]
        want_p = getattr(tr.splats, f).detach().cpu().numpy().ravel()
        # Adam's first steps move every parameter by ~lr * sign(g): entries whose gradient is atomics-order
        # noise around zero may move the other way, so bound the fraction of differing entries
        d = np.abs(got_p - want_p)
        frac = float(np.mean(d > 1e-6 + 1e-5 * np.abs(want_p)))
        assert frac < 1e-3, (f, frac, float(d.max()))
        if not sharded:
            got_g = grads[offs[f]:offs[f] + sizes[f]].astype(np.float64)
            want_g = getattr(tr.grads, f).detach().cpu().numpy().ravel().astype(np.float64)
            rms = float(np.sqrt(np.mean(want_g ** 2))) + 1e-30
            bad = np.abs(got_g - want_g) > 1e-3 * np.abs(want_g) + 1e-4 * rms
            assert int(bad.sum()) == 0, (f, int(bad.sum()))
