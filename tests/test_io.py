"""CSM1 / CTT1 containers against the reference's
own writer (oracle/_ref: io.cpp compiled where it lies): byte-identical
files, round trips, and the reference's error behaviour."""
import os
import struct

import numpy as np
import pytest

import pyoracle
from paper_2511_12235_b200 import TEST_GEOMETRIES, CtsmError
from paper_2511_12235_b200 import io as cio
from paper_2511_12235_b200.projector import _meta

needs_ref = pytest.mark.skipif(not pyoracle.available("ref_cr"), reason="oracle/_ref not built")


@needs_ref
def test_ctt1_bytes_match_reference(tmp_path):
    ref = pyoracle.load("ref_cr")
    data = np.random.default_rng(1).normal(size=(3, 4, 5))
    a, b = tmp_path / "a.ctt", tmp_path / "b.ctt"
    cio.write_tensor(a, data.shape, data)
    ref.write_tensor(str(b), data.shape, data)
    assert a.read_bytes() == b.read_bytes()
    out, dims = cio.read_tensor(b)
    assert dims == [3, 4, 5] and np.array_equal(out, data.ravel())


def test_ctt1_errors(tmp_path):
    p = tmp_path / "x.ctt"
    with pytest.raises(CtsmError) as e:
        cio.write_tensor(p, [], np.zeros(0))
    assert e.value.code == "InvalidSpec"
    with pytest.raises(CtsmError) as e:
        cio.write_tensor(p, [2, 2], np.zeros(3))
    assert e.value.code == "DimensionMismatch"
    p.write_bytes(b"NOPE" + b"\0" * 16)
    with pytest.raises(CtsmError) as e:
        cio.read_tensor(p)
    assert e.value.code == "IoFailure"
    p.write_bytes(b"CTT1" + struct.pack("<I", 9))
    with pytest.raises(CtsmError) as e:
        cio.read_tensor(p)
    assert e.value.code == "IoFailure"
    with pytest.raises(CtsmError) as e:
        cio.read_tensor(tmp_path / "missing.ctt")
    assert e.value.code == "IoFailure"


def test_csm1_header_errors(tmp_path):
    p = tmp_path / "m.csm"
    p.write_bytes(b"CSMX" + b"\0" * 32)
    with pytest.raises(CtsmError) as e:
        cio.read_matrix(p)
    assert e.value.code == "IoFailure"
    p.write_bytes(b"CSM1" + struct.pack("<4Q", 1, 1 << 32, 0, 0))
    with pytest.raises(CtsmError) as e:
        cio.read_matrix(p)
    assert e.value.code == "TooLarge"


@needs_ref
@pytest.mark.parametrize("name", ["proj2d", "cone3d"])
def test_meta_matches_reference(name, tmp_path):
    """projector.cpp:191-199: the metadata block of the device-built matrix."""
    ref = pyoracle.load("ref_cr")
    g = TEST_GEOMETRIES[name]
    p = tmp_path / "r.csm"
    ref.write_matrix(g, str(p))
    _, _, meta = ref.read_matrix(str(p))
    assert _meta(g, "consistent", 1) == meta


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("name", ["proj2d", "proj3d", "cone3d"])
def test_csm1_device_roundtrip_and_bytes(name, tmp_path):
    import torch
    from paper_2511_12235_b200 import build_system_matrix
    ref = pyoracle.load("ref_cr")
    g = TEST_GEOMETRIES[name]
    w = build_system_matrix(g)
    ours, theirs = tmp_path / "ours.csm", tmp_path / "ref.csm"
    cio.write_matrix(ours, w)
    ref.write_matrix(g, str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()  # bit-exact CSR + same container
    for path in (ours, theirs):
        r = cio.read_matrix(path)
        assert (r.n_rows, r.n_cols, r.meta) == (w.n_rows, w.n_cols, w.meta)
        assert torch.equal(r.row_start, w.row_start)
        assert torch.equal(r.col, w.col)
        assert torch.equal(r.val, w.val)


@pytest.mark.gpu
def test_csm1_reader_rejects_corruption(tmp_path):
    from paper_2511_12235_b200 import build_system_matrix
    g = TEST_GEOMETRIES["proj2d"]
    w = build_system_matrix(g)
    good = tmp_path / "g.csm"
    cio.write_matrix(good, w)
    raw = bytearray(good.read_bytes())
    hdr = 4 + 32 + len(w.meta.encode())
    rs_bytes = 8 * (w.n_rows + 1)
    # a column index out of range
    bad = bytearray(raw)
    struct.pack_into("<Q", bad, hdr + rs_bytes, w.n_cols + 5)
    (tmp_path / "c.csm").write_bytes(bad)
    # decreasing row offsets
    bad2 = bytearray(raw)
    struct.pack_into("<Q", bad2, hdr + 8 * 20, 1 << 40)
    (tmp_path / "d.csm").write_bytes(bad2)
    # truncated payload
    (tmp_path / "t.csm").write_bytes(bytes(raw[:-100]))
    for name in ("c.csm", "d.csm", "t.csm"):
        with pytest.raises(CtsmError) as e:
            cio.read_matrix(tmp_path / name)
        assert e.value.code == "IoFailure", name
