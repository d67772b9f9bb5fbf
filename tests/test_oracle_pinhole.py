"""Pin the oracle's perspective (pinhole) extension, which has no reference
implementation: naive-vs-tiled equivalence with thresholds
disabled and analytic-vs-finite-difference gradients
(reference.hpp:66-105 pattern), excluding kinks."""
import numpy as np
import pytest

from parity import O


def _tiny(seed, n, K=6):
    import paper_2412_12734_b200.scenes as sc

    arrays = sc.generate(O.MODE_PINHOLE, K, n, seed, mean_lo=-0.6, mean_hi=0.6, scale_lo=0.15, scale_hi=0.4)
    spec = sc.look_at((0.3, -0.2, -3.0), (0.0, 0.0, 0.0), 16, 16, 20.0, 22.0, 8.0, 8.0)
    cam = O.Cam.from_spec(spec)
    cam.background = (0.2, 0.5, 0.1)
    return arrays, cam


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("n", [1, 2, 4])
def test_pinhole_tiled_equals_naive(seed, n):
    arrays, cam = _tiny(seed, n)
    scene = O.Scene64(arrays, n)
    cfg = O.Cfg(tile_size=4, cutoff_radius=0.0, alpha_skip=0.0, early_stop=0.0, threads=2)
    b = O.build_binning(scene, cam, cfg)
    f = O.render_forward(scene, cam, cfg, b)
    color, trans = O.render_naive(scene, cam)
    np.testing.assert_allclose(f["color"], color, atol=1e-12)
    np.testing.assert_allclose(f["trans"], trans, atol=1e-12)


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("n", [1, 2, 4])
def test_pinhole_gradient_matches_fd(seed, n):
    """Analytic backward vs central FD of a linear image loss; entries whose FD
    stencil crosses a kink (kink slack > 0) are excluded, as SPEC.md:316 does."""
    arrays, cam = _tiny(seed, n)
    scene = O.Scene64(arrays, n)
    cfg = O.Cfg(tile_size=4, cutoff_radius=0.0, alpha_skip=0.0, early_stop=0.0, threads=2)
    b = O.build_binning(scene, cam, cfg)
    f = O.render_forward(scene, cam, cfg, b)
    w = np.random.default_rng(100 + seed).standard_normal((cam.height, cam.width, 3))
    g, mag, slack = O.render_backward(scene, cam, cfg, b, f, w, kink=(2e-5, 1e-3, 2e-3, 1e-3))
    fd = O.gradient_fd(scene, cam, w, 1e-6)
    for k in ("position", "quat", "log_scale", "opacity_logit", "grid"):
        ok = slack[k] == 0
        err = np.abs(g[k] - fd[k])[ok]
        tol = 1e-5 + 1e-3 * np.abs(fd[k])[ok]
        assert np.all(err <= tol), (k, float((err / tol).max()))


def test_pinhole_depth_key_is_camera_z_rounded_to_fp32():
    arrays, cam = _tiny(0, 2, K=20)
    scene = O.Scene64(arrays, 2)
    depth, rect = O.project(scene, cam, O.Cfg(tile_size=4))
    R = np.asarray(cam.rot); t = np.asarray(cam.trans)
    z = arrays["position"].astype(np.float64) @ R[2] + t[2]
    np.testing.assert_array_equal(depth, z.astype(np.float32).astype(np.float64))


def test_pinhole_near_plane_cull_and_behind_camera():
    arrays, cam = _tiny(1, 2, K=4)
    arrays = {k: (None if v is None else v.copy()) for k, v in arrays.items()}
    arrays["position"][0] = (0.0, 0.0, -3.5)  # behind the camera (eye at z=-3)
    arrays["position"][1] = (0.0, 0.0, -2.995)  # in front of the camera but closer than the near plane
    scene = O.Scene64(arrays, 2)
    depth, rect = O.project(scene, cam, O.Cfg(tile_size=4))
    assert rect[0, 0] == -1 and rect[1, 0] == -1


def test_pinhole_intersection_matches_plane_geometry():
    """(u, v) from the Cramer solution equal the plane coordinates of the ray hit."""
    import ctypes as C

    L = O.oracle_lib()
    cam = O.Cam(O.MODE_PINHOLE, 64, 48, (0, 0, 0), 50.0, 60.0, 31.0, 23.5, np.eye(3), np.array([0.0, 0.0, 5.0]))
    mean = np.array([0.2, -0.1, 0.3]); q = np.array([0.9, 0.2, -0.3, 0.1]); ls = np.log([0.3, 0.7])
    u, v = C.c_double(), C.c_double()
    px, py = 35.5, 20.5
    cc = cam.to_c()
    ok = L.orc_intersect_pinhole(C.byref(cc), mean.ctypes.data, q.ctypes.data, ls.ctypes.data, px, py, C.byref(u),
                                 C.byref(v))
    assert ok
    qn = q / np.linalg.norm(q)
    w, x, y, z = qn
    tu = np.array([1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y)])
    tv = np.array([2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x)])
    P = mean + np.array([0.0, 0.0, 5.0]) + 0.3 * tu * u.value + 0.7 * tv * v.value  # camera space
    np.testing.assert_allclose([P[0] / P[2] * 50.0 + 31.0, P[1] / P[2] * 60.0 + 23.5], [px, py], atol=1e-9)
