"""Regenerate the golden fixtures from the COMPILED REFERENCE (oracle/_ref/libgbil_ref.so).

Run in the build container, where /root/reference exists:
    make -C oracle && python tests/golden/make_golden.py

Writes (small, committed):
  ortho_cases.npz -- seeded ortho scenes (fp32 inputs) with the reference's
                     build_binning CSR, render_forward outputs and
                     render_backward gradients for a fixed +-1 image_grad
  naive_fd.npz    -- reference render_naive + gradient_fd on a tiny scene
  rng.npz         -- reference Rng uniform()/normal() streams
  kat.json        -- SPEC known-answer examples evaluated by the reference
  ref_k9_n3.gbil  -- a GBIL v1 splat file written by the reference's save_splats
  diag_cases.npz  -- the reference's downsample_grid on seeded grids (n, levels sweep) and its
                     randomize_colors stream
  fit_cases.npz   -- the reference's fit() (train.hpp:174-219) on small seeded targets (MSE and
                     MSE + SSIM) and its ssim / ssim_with_gradient / psnr on seeded image pairs
The fixtures travel to the GPU box; nothing there reads /root/reference.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
import paper_2412_12734_b200.scenes as sc  # noqa: E402

# (name, K, n, W, H, seed, scale_lo, scale_hi, tile, cutoff, skip, early_stop, background)
CASES = [
    ("n1", 150, 1, 64, 48, 101, 0.7, 6.0, 16, 3.0, 1 / 255, 1e-4, (0.0, 0.0, 0.0)),
    ("n2", 150, 2, 64, 48, 102, 0.7, 6.0, 16, 3.0, 1 / 255, 1e-4, (0.2, 0.4, 0.6)),
    ("n3", 120, 3, 50, 37, 103, 0.7, 6.0, 16, 3.0, 1 / 255, 1e-4, (0.1, 0.1, 0.1)),
    ("n4", 150, 4, 64, 48, 104, 0.7, 6.0, 16, 3.0, 1 / 255, 1e-4, (1.0, 1.0, 1.0)),
    ("n8", 150, 8, 64, 48, 105, 0.7, 6.0, 16, 3.0, 1 / 255, 1e-4, (0.0, 0.5, 0.0)),
    ("n4_tile5", 120, 4, 41, 29, 106, 0.7, 5.0, 5, 3.0, 1 / 255, 1e-4, (0.3, 0.3, 0.3)),
    ("n4_nothresh", 60, 4, 32, 24, 107, 1.0, 5.0, 16, 0.0, 0.0, 0.0, (0.5, 0.2, 0.9)),
    ("n2_dense", 400, 2, 48, 32, 108, 1.0, 10.0, 8, 3.0, 1 / 255, 1e-4, (0.0, 0.0, 0.0)),
]


def ortho_cases():
    out = {}
    for name, K, n, W, H, seed, lo, hi, ts, cut, skip, es, bg in CASES:
        arr = sc.generate(O.MODE_ORTHO, K, n, seed, width=W, height=H, scale_lo=lo, scale_hi=hi)
        scene = O.Scene64(arr, n)
        cam = O.Cam(O.MODE_ORTHO, W, H, bg)
        cfg = O.Cfg(tile_size=ts, cutoff_radius=cut, alpha_skip=skip, early_stop=es, threads=3)
        ig = np.random.default_rng(seed).choice(np.array([-1.0, 0.0, 1.0]), size=(H, W, 3))
        r = O.ref_render(scene, cam, cfg, ig)
        meta = dict(K=K, n=n, W=W, H=H, tile=ts, cutoff=cut, skip=skip, early_stop=es, bg=list(bg))
        out[f"{name}/meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
        for k in ("position", "depth_key", "theta", "log_scale", "opacity_logit", "grid"):
            out[f"{name}/in_{k}"] = arr[k]
        out[f"{name}/image_grad"] = ig.astype(np.int8)
        for k in ("offsets", "values", "color", "trans", "last"):
            out[f"{name}/{k}"] = r[k]
        for k, v in r["grads"].items():
            out[f"{name}/g_{k}"] = v
    np.savez_compressed(os.path.join(HERE, "ortho_cases.npz"), **out)


def naive_fd():
    arr = sc.generate(O.MODE_ORTHO, 5, 2, 7, width=16, height=16, scale_lo=1.5, scale_hi=4.0)
    scene = O.Scene64(arr, 2)
    cam = O.Cam(O.MODE_ORTHO, 16, 16, (0.1, 0.2, 0.3))
    w = np.random.default_rng(7).standard_normal((16, 16, 3))
    color, trans = O.ref_render_naive(scene, cam)
    g = O.ref_gradient_fd(scene, cam, w, 1e-6)
    out = {f"in_{k}": arr[k] for k in ("position", "depth_key", "theta", "log_scale", "opacity_logit", "grid")}
    out.update(weights=w, color=color, trans=trans, **{f"g_{k}": v for k, v in g.items() if v is not None})
    np.savez_compressed(os.path.join(HERE, "naive_fd.npz"), **out)


def rng_streams():
    L = O.ref_lib()
    out = {}
    for seed in (0, 1, 2, 12345, 2 ** 63 + 5):
        u = np.zeros(1000)
        L.ref_rng_uniform(seed, 1000, u.ctypes.data)
        nrm = np.zeros(1001)
        L.ref_rng_normal(seed, 1001, 0.0, 1.0, nrm.ctypes.data)
        out[f"uniform_{seed}"] = u
        out[f"normal_{seed}"] = nrm
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **out)


def kat():
    import ctypes as C

    L = O.ref_lib()
    res = {}

    def uv(u, v, n, s):
        iu, iv, fu, fv = C.c_int32(), C.c_int32(), C.c_double(), C.c_double()
        L.ref_uv_to_grid(u, v, n, s, C.byref(iu), C.byref(iv), C.byref(fu), C.byref(fv))
        return [iu.value, iv.value, fu.value, fv.value]

    res["uv_to_grid"] = [[u, v, n, s, uv(u, v, n, s)] for (u, v, n, s) in
                         [(-0.5, -0.5, 4, 0.5), (0.0, 0.0, 2, 0.5), (5.0, 0.0, 4, 0.5), (0.13, -0.31, 8, 0.5),
                          (-7.0, 7.0, 8, 2.0), (0.25, 0.25, 1, 0.5)]]
    grid2 = np.array([0, 0, 0, 0, 0, 1, 1, 0, 0, 1, 0, 1], np.float64)  # C[0,0],C[0,1],C[1,0],C[1,1]

    def bil(u, v, n, s, g):
        c = np.zeros(3)
        L.ref_bilinear(u, v, n, s, g.ctypes.data, c.ctypes.data)
        return c.tolist()

    res["bilinear"] = [[u, v, bil(u, v, 2, 0.5, grid2)] for (u, v) in [(0.0, 0.0), (5.0, 0.0), (-0.2, 0.3)]]
    rng = np.random.default_rng(3)
    g8 = rng.random(8 * 8 * 3)
    adj = []
    for (u, v) in [(0.11, -0.23), (0.6, 0.1), (-0.49, 0.49), (0.0, 0.0)]:
        ch = np.array([0.3, -0.7, 1.1])
        gg = np.zeros_like(g8)
        uh, vh = C.c_double(), C.c_double()
        L.ref_adj_bilinear(u, v, 8, 0.5, g8.ctypes.data, ch.ctypes.data, gg.ctypes.data, C.byref(uh), C.byref(vh))
        adj.append([u, v, ch.tolist(), gg.tolist(), uh.value, vh.value])
    res["adj_bilinear_grid8"] = g8.tolist()
    res["adj_bilinear"] = adj
    p = np.array([1.0, -2.0, 0.5]); g = np.array([1.0, 1.0, -3.0]); m = np.zeros(3); v = np.zeros(3)
    L.ref_adam_group(p.ctypes.data, g.ctypes.data, m.ctypes.data, v.ctypes.data, 3, 0.1, 0.9, 0.999, 1e-8,
                     1 - 0.9, 1 - 0.999)
    res["adam_first_step"] = dict(p0=[1.0, -2.0, 0.5], g=[1.0, 1.0, -3.0], lr=0.1, p1=p.tolist(), m=m.tolist(),
                                  v=v.tolist())
    with open(os.path.join(HERE, "kat.json"), "w") as fh:
        json.dump(res, fh, indent=1)


def gbil_file():
    """A small v1 splat file written by the reference itself (serialize.hpp:83-90)."""
    arrays = sc.generate(O.MODE_ORTHO, 9, 3, 109, width=40, height=30, scale_lo=0.7, scale_hi=6.0)
    scene = O.Scene64(arrays, 3, 0.375)
    msg = O.ref_save_splats(os.path.join(HERE, "ref_k9_n3.gbil"), scene)
    assert msg == "", msg


FIT_CASES = [  # (name, W, H, K, n, iterations, mse_ssim, seed)
    ("mse_n4", 40, 32, 60, 4, 3, False, 11),
    ("ssim_n2", 36, 30, 50, 2, 3, True, 12),
    ("mse_n1", 24, 20, 30, 1, 2, False, 13),
]


def fit_cases():
    out = {}
    for name, W, H, K, n, iters, ms, seed in FIT_CASES:
        target = sc.uniform_image(1000 + seed, W, H).astype(np.float64)
        res = O.ref_fit(target, K, n, iters, mse_ssim=ms, seed=seed, log_every=1)
        assert not isinstance(res, str), res
        arrays, hist = res
        out[f"{name}/target"] = target.astype(np.float32)
        out[f"{name}/meta"] = np.array([W, H, K, n, iters, int(ms), seed], np.int64)
        out[f"{name}/history"] = hist
        for f, v in arrays.items():
            out[f"{name}/final/{f}"] = v
    rng = np.random.default_rng(5)
    for name, (h, w) in (("img_a", (41, 53)), ("img_b", (11, 11))):
        a = rng.random((h, w, 3)) * 1.2 - 0.1  # exceeds [0,1] so clamping matters
        b = rng.random((h, w, 3))
        a32, b32 = a.astype(np.float32).astype(np.float64), b.astype(np.float32).astype(np.float64)
        v, g = O.ref_ssim(a32, b32, with_grad=True)
        out[f"{name}/a"] = a32.astype(np.float32)
        out[f"{name}/b"] = b32.astype(np.float32)
        out[f"{name}/ssim_clamped"] = np.array(O.ref_ssim(a32, b32))
        out[f"{name}/ssim_raw"] = np.array(v)
        out[f"{name}/ssim_grad"] = g
        out[f"{name}/psnr"] = np.array(O.ref_psnr(a32, b32))
    np.savez_compressed(os.path.join(HERE, "fit_cases.npz"), **out)


DIAG_CASES = [(8, 1), (8, 2), (8, 3), (8, 5), (4, 1), (6, 1), (6, 3), (3, 2), (16, 2), (1, 3), (2, 0)]


def diag_cases():
    out = {}
    rng = np.random.default_rng(9)
    for n, levels in DIAG_CASES:
        grids = rng.random((5, 3 * n * n)).astype(np.float32)
        res = [O.ref_downsample_grid(g.astype(np.float64), n, levels) for g in grids]
        assert not isinstance(res[0], str), res[0]
        out[f"n{n}_l{levels}/in"] = grids
        out[f"n{n}_l{levels}/out"] = np.stack([r[0] for r in res])
        out[f"n{n}_l{levels}/n_out"] = np.array(res[0][1])
    out["randomize/K7_n3_seed5"] = O.ref_randomize_colors(7, 3, 5)
    np.savez_compressed(os.path.join(HERE, "diag_cases.npz"), **out)


if __name__ == "__main__":
    if not O.ref_available():
        O.build()
    ortho_cases()
    naive_fd()
    rng_streams()
    kat()
    gbil_file()
    fit_cases()
    diag_cases()
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
