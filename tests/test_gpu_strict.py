"""Strict gradient parity: the fp64 parity build (-DGB_PARITY_F64) against the fp64 oracle, every entry
within rtol 1e-4 / atol 1e-5 + kink slack, with no cancellation exemption (tests/strict_case.py).

The product library is fp32 and is held to the error-model protocol in test_gpu_parity.py; this build runs
the same kernels in fp64 (summation order is the only difference from the reference's algorithm), so it
separates the kernels' algorithm -- walk order, rewind, adjoint, footprint classes, reductions, Jacobians --
from fp32 rounding and atomics order, the job the reference's ordered reduction does (raster.hpp:293-302,
368-385)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2412_12734_b200", "libgb_raster_f64.so")
OUT = os.path.join(ROOT, "gpurun_out")


@pytest.mark.parametrize("case", ["ortho_n3", "pinhole_small_n8", "configs1", "configs2",
                                  "configs4_1000000_T16_rows8"])
def test_strict_parity_fp64_build(case):
    assert os.path.exists(LIB), "build the parity library (__graft_entry__.build())"
    os.makedirs(OUT, exist_ok=True)
    out = os.path.join(OUT, f"strict_{case}.json")
    env = dict(os.environ, GB_LIB_PATH=LIB)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "strict_case.py"), case, out], env=env,
                       capture_output=True, text=True, timeout=1800)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert os.path.exists(out), r.stderr[-2000:]
    stats = json.load(open(out))
    assert stats["library"] == "libgb_raster_f64.so"
    assert stats["binning"]["offsets_equal"] and stats["binning"]["values_equal"]
    im = stats["image"]
    assert im["color_violations"] == 0 and im["alpha_violations"] == 0 and im["last_rank_mismatch"] == 0, im
    for f, st in stats["grads"].items():
        assert st["strict_violations"] == 0, (f, st)
    assert r.returncode == 0
