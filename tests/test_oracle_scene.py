"""The oracle's own input generator (used by bench.py's reference arm, which must not load the product
library) produces bit-identical inputs to the product's gb_scene_generate / gb_uniform_fill and cameras."""
import numpy as np
import pytest

from oracle import oracle as O


def test_rng_streams_match_reference_golden():
    g = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "rng.npz"))
    for key in g.files:
        kind, seed = key.split("_")[0], int(key.split("_")[1]) if key.count("_") else 0
        if kind == "uniform":
            assert np.array_equal(O.rng_uniform(seed, g[key].size), g[key]), key
        elif kind == "normal":
            assert np.array_equal(O.rng_normal(seed, g[key].size), g[key]), key


def test_config3_inputs_bit_identical_to_product():
    sc = pytest.importorskip("paper_2412_12734_b200.scenes")
    cfg = sc.baseline_config(3, count=5000, n=8)
    ref = cfg.arrays()
    arrays, cams, target = O.config3_inputs(count=5000, n=8)
    for f in ("position", "quat", "log_scale", "opacity_logit", "grid"):
        assert arrays[f].dtype == np.float32
        assert np.array_equal(arrays[f].view(np.uint32), ref[f].view(np.uint32)), f
    assert len(cams) == len(cfg.cameras) == 64
    for a, b in zip(cams, cfg.cameras):
        assert (a.width, a.height, a.fx, a.fy, a.cx, a.cy) == (b.width, b.height, b.fx, b.fy, b.cx, b.cy)
        assert np.array_equal(a.rot, b.rot) and np.array_equal(a.trans, b.trans)
    for v in (0, 5):
        t = target(v)[:16]
        assert np.array_equal(t, cfg.target(v)[:16])


def test_uniform_scene_matches_product():
    sc = pytest.importorskip("paper_2412_12734_b200.scenes")
    ref = sc.generate(sc.MODE_PINHOLE, 777, 4, 3, mean_lo=-2.0, mean_hi=2.0, scale_lo=0.002, scale_hi=0.05)
    got = O.generate_pinhole(777, 4, 3, mean_lo=-2.0, mean_hi=2.0, scale_lo=0.002, scale_hi=0.05)
    for f in ("position", "quat", "log_scale", "opacity_logit", "grid"):
        assert np.array_equal(got[f].view(np.uint32), ref[f].view(np.uint32)), f
