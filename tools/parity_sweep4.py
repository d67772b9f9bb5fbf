"""configs[4] parity sweep at full size (development/evidence tool): every T in {1, 4, 8, 16} x K in
{0.1, 1, 4}M cell through tests/parity.py run_rows (tile-row subset, stride 8) against the fp64 oracle,
one JSON per cell into gpurun_out/parity4_K<K>_T<T>.json (fp32 product) and, with --strict, the fp64
parity build's cells into gpurun_out/strict4_K<K>_T<T>.json (run under GB_LIB_PATH=libgb_raster_f64.so).

    python tools/parity_sweep4.py [--strict]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from parity import O, compare_binning, compare_grads, compare_image, run_rows  # noqa: E402


def main():
    import paper_2412_12734_b200.scenes as sc

    strict = "--strict" in sys.argv
    kink = O.STRICT_KINK if strict else O.DEFAULT_KINK
    out_dir = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out_dir, exist_ok=True)
    for K in (100_000, 1_000_000, 4_000_000):
        for T in (1, 4, 8, 16):
            c = sc.baseline_config(4, count=K, n=T)
            cam = O.Cam.from_spec(c.cameras[0])
            ig = np.random.default_rng(0).choice(np.array([-1.0, 1.0]), size=(cam.height, cam.width, 3))
            gpu, orc, info = run_rows(c.arrays(), O.MODE_PINHOLE, T, cam, O.Cfg(), ig, stride=8, kink=kink)
            st = dict(info=info, binning=compare_binning(gpu, orc), image=compare_image(gpu, orc),
                      grads=compare_grads(gpu, orc), kink=list(kink))
            name = f"{'strict4' if strict else 'parity4'}_K{K}_T{T}.json"
            json.dump(st, open(os.path.join(out_dir, name), "w"), indent=1)
            g = st["grads"]
            ok = (st["binning"]["offsets_equal"] and st["binning"]["values_equal"]
                  and st["image"]["color_violations"] == 0 and st["image"]["alpha_violations"] == 0
                  and st["image"]["last_rank_mismatch"] == 0
                  and all((v["strict_violations"] if strict else v["strict_violations_applicable"] + v["model_violations"]) == 0
                          for v in g.values()))
            print(name, "OK" if ok else "FAIL", info["pairs"], info["subset_pairs"], st["image"]["kink_pixels"],
                  {k: (v["strict_violations"], v["strict_violations_applicable"], v["model_violations"]) for k, v in g.items()},
                  flush=True)
            del gpu, orc


if __name__ == "__main__":
    main()
