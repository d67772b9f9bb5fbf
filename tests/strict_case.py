"""One strict-parity case through the fp64 parity build (test infrastructure; run by tests/test_gpu_strict.py
in a subprocess with GB_LIB_PATH=paper_2412_12734_b200/libgb_raster_f64.so).

The parity build runs the product's K1..K5 code with real = double (gb_internal.cuh, -DGB_PARITY_F64): the
same walk, culls, footprint classes, per-lane/warp reductions and Jacobians, but fp64 arithmetic and fp64
atomics.  It therefore differs from the reference's fp64 algorithm (raster.hpp:198-387) only in summation
order, and every gradient entry is held to rtol 1e-4 / atol 1e-5 plus the oracle's kink slack -- no
cancellation exemption.  Tile lists stay bit-exact and images within tolerance with exact last_rank.

    GB_LIB_PATH=... python tests/strict_case.py <case> <out.json>
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from parity import O, compare_binning, compare_grads, compare_image, run_gpu, run_oracle, run_rows  # noqa: E402


def image_grad(seed, h, w):
    return np.random.default_rng(seed).choice(np.array([-1.0, 1.0]), size=(h, w, 3))


def case(name):
    import paper_2412_12734_b200.scenes as sc

    if name == "ortho_n3":
        W, H = 320, 240
        arrays = sc.generate(O.MODE_ORTHO, 6000, 3, 13, width=W, height=H, scale_lo=0.5, scale_hi=8.0)
        return arrays, O.MODE_ORTHO, 3, O.Cam(O.MODE_ORTHO, W, H, (0.1, 0.3, 0.7)), None
    if name == "pinhole_small_n8":
        c = sc.baseline_config(0, count=20_000, n=8)
        return c.arrays(), O.MODE_PINHOLE, 8, O.Cam.from_spec(c.cameras[0]), None
    if name in ("configs1", "configs2"):
        c = sc.baseline_config(int(name[-1]))
        return c.arrays(), O.MODE_PINHOLE, c.n, O.Cam.from_spec(c.cameras[0]), None
    if name.startswith("configs4_"):  # configs4_<K>_T<n>_rows<stride>
        _, k, t, r = name.split("_")
        c = sc.baseline_config(4, count=int(k), n=int(t[1:]))
        return c.arrays(), O.MODE_PINHOLE, c.n, O.Cam.from_spec(c.cameras[0]), int(r[4:])
    raise ValueError(name)


def main():
    name, out = sys.argv[1], sys.argv[2]
    arrays, mode, n, cam, stride = case(name)
    ig = image_grad(0, cam.height, cam.width)
    cfg = O.Cfg()
    # decision kinks only: the parity build evaluates (u, v) in fp64, so no fp32 (u, v) error is propagated
    if stride:
        gpu, orc, info = run_rows(arrays, mode, n, cam, cfg, ig, stride=stride, kink=O.STRICT_KINK)
    else:
        gpu = run_gpu(arrays, mode, n, cam, cfg, ig)
        orc = run_oracle(arrays, n, cam, cfg, ig, kink=O.STRICT_KINK)
        info = {}
    import paper_2412_12734_b200._lib as L

    stats = dict(case=name, library=os.path.basename(L.LIB_PATH), info=info, binning=compare_binning(gpu, orc),
                 image=compare_image(gpu, orc), grads=compare_grads(gpu, orc))
    with open(out, "w") as fh:
        json.dump(stats, fh, indent=1)
    ok = (stats["binning"]["offsets_equal"] and stats["binning"]["values_equal"]
          and stats["image"]["color_violations"] == 0 and stats["image"]["alpha_violations"] == 0
          and stats["image"]["last_rank_mismatch"] == 0
          and all(st["strict_violations"] == 0 for st in stats["grads"].values()))
    print(name, "strict", {f: st["strict_violations"] for f, st in stats["grads"].items()},
          "exempt-if-fp32", {f: st["cancellation_exempt"] for f, st in stats["grads"].items()}, stats["image"])
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
