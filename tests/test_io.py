"""On-disk formats next to the path, host only (no GPU):
.flo against the reference's own read_flo / write_flo (oracle/_ref) both ways; .stnt raw
tensors pinned to the byte layout video_io.cpp:52-117 writes (the reference's video_io.cpp
needs libpng, absent here, so it is not run) plus round trips and every header error."""
import ctypes as C
import os
import struct

import numpy as np
import pytest

from oracle.oracle import Checker, have_reference
from paper_2309_16849_b200 import snls as S


def test_flo_round_trip_and_reference_interop(tmp_path):
    P = Checker("port")
    h, w = 7, 9
    flow = P.uniform(5, -20, 20, h * w * 2).reshape(h, w, 2).astype(np.float32)
    ours = str(tmp_path / "ours.flo")
    S.write_flo(ours, flow)
    assert np.array_equal(S.read_flo(ours), flow)
    raw = open(ours, "rb").read()
    assert struct.unpack("<fii", raw[:12]) == (202021.25, w, h)
    assert struct.unpack("<ff", raw[12:20]) == (flow[0, 0, 1], flow[0, 0, 0])  # (u, v) = (dx, dy)
    if not have_reference():
        pytest.skip("oracle/_ref not built")
    R = Checker("reference")
    got = np.zeros((h, w, 2))
    R.lib.ref_read_flo.argtypes = [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_double)]
    assert R.lib.ref_read_flo(ours.encode(), h, w, got.ctypes.data_as(C.POINTER(C.c_double))) == 0
    assert np.array_equal(got, flow.astype(np.float64))
    theirs = str(tmp_path / "ref.flo")
    f64 = np.ascontiguousarray(flow, np.float64)
    R.lib.ref_write_flo.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_double), C.c_char_p]
    assert R.lib.ref_write_flo(h, w, f64.ctypes.data_as(C.POINTER(C.c_double)), theirs.encode()) == 0
    assert open(theirs, "rb").read() == raw
    assert np.array_equal(S.read_flo(theirs), flow)


def test_flo_errors(tmp_path):
    bad = tmp_path / "bad.flo"
    bad.write_bytes(struct.pack("<fii", 1.0, 2, 2) + b"\0" * 32)
    with pytest.raises(S.IoError, match="bad magic"):
        S.read_flo(str(bad))
    bad.write_bytes(struct.pack("<fii", 202021.25, 2, 2) + b"\0" * 8)
    with pytest.raises(S.IoError, match="truncated payload"):
        S.read_flo(str(bad))
    bad.write_bytes(struct.pack("<fii", 202021.25, 0, 2))
    with pytest.raises(S.IoError, match="nonsensical dimensions 0x2"):
        S.read_flo(str(bad))
    with pytest.raises(S.IoError, match="cannot open"):
        S.read_flo(str(tmp_path / "missing.flo"))
    nan = tmp_path / "nan.flo"
    nan.write_bytes(struct.pack("<fii", 202021.25, 1, 1) + struct.pack("<ff", float("nan"), 0.0))
    with pytest.raises(S.DomainError, match="non-finite"):
        S.read_flo(str(nan))


@pytest.mark.parametrize("width", [4, 8])
def test_raw_layout_round_trip_and_errors(tmp_path, width):
    P = Checker("port")
    v = P.uniform(9, -3, 3, 2 * 3 * 4 * 5).reshape(2, 3, 4, 5).astype(np.float32)
    path = str(tmp_path / "v.stnt")
    S.write_raw(path, v, width)
    raw = open(path, "rb").read()
    # video_io.cpp:92-117: magic, u32 t h w f, width byte, little-endian payload
    assert raw[:4] == b"STNT" and struct.unpack("<IIII", raw[4:20]) == (2, 3, 4, 5) and raw[20] == width
    fmt = "<" + ("f" if width == 4 else "d") * v.size
    assert np.array_equal(np.array(struct.unpack(fmt, raw[21:])), v.reshape(-1).astype(np.float64))
    assert np.array_equal(S.read_raw(path), v)
    for payload, msg in ((raw[:20], "truncated header"), (b"XXXX" + raw[4:], "bad magic"),
                         (raw[:20] + bytes([3]) + raw[21:], "element width must be 4 or 8"),
                         (raw[:4] + struct.pack("<I", 0) + raw[8:], "zero extent in header"),
                         (raw + b"\0", "payload size does not match header")):
        bad = tmp_path / "bad.stnt"
        bad.write_bytes(payload)
        with pytest.raises(S.IoError, match=msg):
            S.read_raw(str(bad))
