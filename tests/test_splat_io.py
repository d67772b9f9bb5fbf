"""GBIL splat files (serialize.hpp:15-124) through the C-ABI.

CPU: header and structure validation (gb_splats_file_info) on the reference-written
fixture and on corrupted copies; every error message must equal the reference's own
(checked against the compiled reference where it exists, else against the pinned
strings).  GPU: load of the reference fixture is bit-exact, save reproduces its bytes,
pinhole (version 2) and chunk-spanning files round-trip exactly.
"""
import os
import shutil
import struct

import numpy as np
import pytest

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "ref_k9_n3.gbil")


def _scene():
    import paper_2412_12734_b200.scenes as sc

    return sc.generate(O.MODE_ORTHO, 9, 3, 109, width=40, height=30, scale_lo=0.7, scale_hi=6.0)


def _info_error(path):
    import paper_2412_12734_b200 as gb

    with pytest.raises(gb.SplatIoError) as e:
        gb.file_info(path)
    return str(e.value).split(": status 7: ", 1)[1]


def test_file_info_of_reference_file():
    import paper_2412_12734_b200 as gb

    info = gb.file_info(GOLDEN)
    assert (info.version, info.mode, info.count, info.n) == (1, O.MODE_ORTHO, 9, 3)
    assert info.sigma == np.float32(0.375)


def _corrupt(tmp_path, name, mutate):
    p = str(tmp_path / name)
    shutil.copy(GOLDEN, p)
    data = bytearray(open(p, "rb").read())
    data = mutate(data)
    open(p, "wb").write(bytes(data))
    return p


CORRUPTIONS = [
    ("magic", lambda d: b"GBIX" + d[4:], "bad splat file: wrong magic"),
    ("short_magic", lambda d: d[:3], "bad splat file: wrong magic"),
    ("header", lambda d: d[:14], "bad splat file: truncated header"),
    ("version", lambda d: d[:4] + struct.pack("<I", 99) + d[8:], "unsupported splat file version 99"),
    ("n0", lambda d: d[:12] + struct.pack("<I", 0) + d[16:], "bad splat file: invalid grid config"),
    ("sigma", lambda d: d[:16] + struct.pack("<f", 0.0) + d[20:], "bad splat file: invalid grid config"),
    ("records", lambda d: d[:20 + 136 * 4 + 17], "bad splat file: truncated at record 4"),
    ("last_record", lambda d: d[:-1], "bad splat file: truncated at record 8"),
]


@pytest.mark.parametrize("name,mutate,expected", CORRUPTIONS, ids=[c[0] for c in CORRUPTIONS])
def test_corrupt_files_match_reference_messages(tmp_path, name, mutate, expected):
    p = _corrupt(tmp_path, name, mutate)
    assert _info_error(p) == expected
    if O.ref_available():  # the pinned strings are the reference's own
        assert O.ref_load_splats(p) == expected


def test_missing_file():
    p = "/nonexistent/x.gbil"
    assert _info_error(p) == f"cannot open splat file: {p}"
    if O.ref_available():
        assert O.ref_load_splats(p) == f"cannot open splat file: {p}"


@pytest.mark.skipif(not O.ref_available(), reason="compiled reference not present (GPU box)")
def test_golden_fixture_is_what_the_reference_writes(tmp_path):
    p = str(tmp_path / "again.gbil")
    assert O.ref_save_splats(p, O.Scene64(_scene(), 3, 0.375)) == ""
    assert open(p, "rb").read() == open(GOLDEN, "rb").read()


@pytest.mark.gpu
def test_load_reference_file_bit_exact():
    import paper_2412_12734_b200 as gb

    s = gb.load_splats(GOLDEN)
    ref = _scene()
    assert s.mode == O.MODE_ORTHO and s.count == 9 and s.grid_config.n == 3
    for f, v in s.tensors().items():
        np.testing.assert_array_equal(v.cpu().numpy().reshape(ref[f].shape), ref[f], err_msg=f)


@pytest.mark.gpu
def test_save_reproduces_reference_bytes(tmp_path):
    import paper_2412_12734_b200 as gb

    s = gb.SplatSet.from_numpy(O.MODE_ORTHO, gb.ColorGridConfig(3, 0.375), **_scene())
    p = str(tmp_path / "ours.gbil")
    gb.save_splats(p, s)
    assert open(p, "rb").read() == open(GOLDEN, "rb").read()


@pytest.mark.gpu
@pytest.mark.parametrize("K,n", [(5, 1), (300_000, 8)])
def test_pinhole_round_trip(tmp_path, K, n):
    import torch

    import paper_2412_12734_b200 as gb
    import paper_2412_12734_b200.scenes as sc

    arrays = sc.generate(O.MODE_PINHOLE, K, n, 7)
    s = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(n), **arrays)
    p = str(tmp_path / "pin.gbil")
    gb.save_splats(p, s)  # 300k x 8x8: 239 MB, spans many 16 MB staging chunks
    info = gb.file_info(p)
    assert (info.version, info.mode, info.count, info.n) == (2, O.MODE_PINHOLE, K, n)
    assert os.path.getsize(p) == 20 + K * (10 + 3 * n * n) * 4
    t = gb.load_splats(p)
    for f, v in s.tensors().items():
        assert torch.equal(t.tensors()[f], v), f
    if K > 100:  # truncated mid-file: the loader names the first incomplete record
        with open(p, "r+b") as fh:
            fh.truncate(20 + 1234 * (10 + 3 * n * n) * 4 + 5)
        with pytest.raises(gb.SplatIoError, match="truncated at record 1234"):
            gb.load_splats(p)
