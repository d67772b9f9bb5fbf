"""bench.py's CPU reference arm samples a view in bands of tile rows: the bands partition the binning."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_band_binning_partitions_the_lists():
    import bench

    rng = np.random.default_rng(0)
    tx, ty = 7, 11
    lens = rng.integers(0, 5, tx * ty)
    offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    values = rng.integers(0, 1000, offsets[-1]).astype(np.int32)
    seen = np.zeros(tx * ty, np.int64)
    rows = []
    for band in range(8):
        (off, val, dims), r0, r1 = bench.band_binning((offsets, values, (tx, ty)), band, 8)
        assert dims == (tx, ty) and off[0] == 0 and len(off) == tx * ty + 1 and off[-1] == len(val)
        rows.append((r0, r1))
        for t in range(tx * ty):
            n = off[t + 1] - off[t]
            if n:
                assert r0 <= t // tx < r1
                np.testing.assert_array_equal(val[off[t]:off[t + 1]], values[offsets[t]:offsets[t + 1]])
                seen[t] += n
    np.testing.assert_array_equal(seen, lens)
    assert rows[0][0] == 0 and rows[-1][1] == ty and all(rows[i][1] == rows[i + 1][0] for i in range(7))
