"""The reference's file formats (io.hpp:52-183): byte layout, round trips, errors."""
import io
import struct

import numpy as np
import pytest

import paper_1412_1885_b200 as P
from paper_1412_1885_b200 import io as tio


def test_dten_byte_layout_and_round_trip(tmp_path):
    a = np.arange(24, dtype=np.float64).reshape((2, 3, 4), order="F")
    buf = io.BytesIO()
    tio.write_dten(buf, a)
    raw = buf.getvalue()
    assert raw[:4] == b"DTEN" and struct.unpack("<IIIII", raw[4:24]) == (1, 3, 2, 3, 4)
    assert np.frombuffer(raw[24:], "<f8").tolist() == list(range(24))  # column-major payload
    t = tio.read_dten(io.BytesIO(raw))
    assert t.shape == (2, 3, 4) and np.array_equal(t.data, a.ravel(order="F"))
    p = tmp_path / "y.dten"
    tio.save_dten(p, t)
    t32 = tio.load_dten(p, dtype=np.float32)
    assert t32.data.dtype == np.float32 and np.array_equal(t32.data, a.ravel(order="F").astype(np.float32))


def test_tkr_and_cpm_round_trip(tmp_path, O):
    g, us = O.rand_tucker_2i(O.gen_tucker((12, 10, 8), (2, 3, 2), (1, 2)), (2, 3, 2), 1, (3, 0))
    m = P.TuckerModel(g, us, g.shape)
    tio.save_tkr(tmp_path / "m.tkr", m)
    r = tio.load_tkr(tmp_path / "m.tkr")
    assert r.core_shape == g.shape and np.array_equal(r.core, g)
    assert all(np.array_equal(a, b) for a, b in zip(r.factors, us))
    raw = (tmp_path / "m.tkr").read_bytes()
    assert raw[:4] == b"TKRM" and struct.unpack("<II", raw[4:12]) == (1, 3)
    fs = [O.gaussian_matrix(d, 4, (5, n)) for n, d in enumerate((7, 6, 5))]
    tio.save_cpm(tmp_path / "c.cpm", P.CpModel(fs))
    c = tio.load_cpm(tmp_path / "c.cpm")
    assert all(np.array_equal(a, b) for a, b in zip(c.factors, fs))
    raw = (tmp_path / "c.cpm").read_bytes()
    assert raw[:4] == b"CPMD" and struct.unpack("<IIIIII", raw[4:28]) == (1, 3, 4, 7, 6, 5)


@pytest.mark.parametrize("data,msg", [
    (b"XTEN" + struct.pack("<II", 1, 1), "bad magic for tensor file"),
    (b"DTEN" + struct.pack("<II", 2, 1), "unsupported tensor file version"),
    (b"DTEN" + struct.pack("<III", 1, 1, 4) + b"\0" * 8, "unexpected end of file"),
    (b"DTEN" + struct.pack("<II", 1, 0), "tensor order must be positive"),
])
def test_dten_errors_match_reference(data, msg):
    with pytest.raises(tio.TenkitIOError, match="tenkit io: " + msg):
        tio.read_dten(io.BytesIO(data))


def test_missing_file():
    with pytest.raises(tio.TenkitIOError, match="cannot open"):
        tio.load_tkr("/nonexistent/x.tkr")
