"""configs[4] cells at their full size (1600x1064, means U[-2,2]^3, scales log-U[0.002, 0.05]) against the
fp64 oracle, on a tile-row subset (tests/parity.py run_rows): every pair of the binning is
compared bit-exactly, and the forward and backward on every 8th tile row (plus the ragged last row), where
the deep-stack rewind (raster.hpp:324-364, T /= 1 - alpha at :333) and the T = 16 adjoint
(texture.hpp:77-111) are most stressed.  Production fp32 library, error-model protocol as
test_gpu_parity.py."""
import json
import os

import numpy as np
import pytest

from parity import O, compare_binning, compare_grads, compare_image, run_rows

pytestmark = pytest.mark.gpu

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


@pytest.mark.parametrize("K,T", [(4_000_000, 16), (4_000_000, 1), (1_000_000, 4)])
def test_configs4_cell_at_size(K, T):
    import paper_2412_12734_b200.scenes as sc

    c = sc.baseline_config(4, count=K, n=T)
    cam = O.Cam.from_spec(c.cameras[0])
    ig = np.random.default_rng(0).choice(np.array([-1.0, 1.0]), size=(cam.height, cam.width, 3))
    gpu, orc, info = run_rows(c.arrays(), O.MODE_PINHOLE, T, cam, O.Cfg(), ig, stride=8)
    stats = dict(info=info, binning=compare_binning(gpu, orc), image=compare_image(gpu, orc),
                 grads=compare_grads(gpu, orc))
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"parity_configs4_K{K}_T{T}.json"), "w") as fh:
        json.dump(stats, fh, indent=1)
    print(json.dumps(stats)[:3000])
    assert stats["binning"]["offsets_equal"] and stats["binning"]["values_equal"]
    assert all(v == 0 for v in info["gpu_nonzero_outside_subset"].values()), info
    im = stats["image"]
    assert im["color_violations"] == 0 and im["alpha_violations"] == 0 and im["last_rank_mismatch"] == 0, im
    for f, st in stats["grads"].items():
        assert st["strict_violations_applicable"] == 0, (f, st)
        assert st["model_violations"] == 0, (f, st)
