"""CGH1 hologram files (image_io.cpp:220-278; format SPEC.md:309): host I/O of
the C ABI, byte layout pinned by the spec (no GPU needed)."""
import struct

import numpy as np
import pytest

from paper_2211_09938_b200 import _lib, stages


def test_cgh1_round_trip_and_layout(tmp_path):
    rng = np.random.default_rng(0)
    n = 16
    plane = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))).astype(np.complex64)
    p = tmp_path / "h.cgh"
    stages.write_cgh1(p, plane, (532e-9, 8e-6, 0.2))
    raw = p.read_bytes()
    assert len(raw) == 34 + n * n * 8
    magic, version, size, wl, pitch, z = struct.unpack("<4sHIddd", raw[:34])
    assert (magic, version, size, wl, pitch, z) == (b"CGH1", 1, n, 532e-9, 8e-6, 0.2)
    assert raw[34:] == plane.tobytes()  # interleaved f32 (re, im), row-major
    back, scene = stages.read_cgh1(p)
    assert np.array_equal(back, plane) and scene == (532e-9, 8e-6, 0.2)


def test_cgh1_errors(tmp_path):
    plane = np.zeros((8, 8), np.complex64)
    p = tmp_path / "h.cgh"
    stages.write_cgh1(p, plane, (532e-9, 8e-6, 0.2))
    raw = p.read_bytes()
    (tmp_path / "trunc.cgh").write_bytes(raw[: len(raw) // 2])
    (tmp_path / "magic.cgh").write_bytes(b"XXXXnotahologram")
    bad = bytearray(raw)
    bad[34:38] = struct.pack("<f", float("nan"))
    (tmp_path / "nan.cgh").write_bytes(bytes(bad))
    with pytest.raises(_lib.IoError):
        stages.read_cgh1(tmp_path / "trunc.cgh")
    with pytest.raises(_lib.IoError):
        stages.read_cgh1(tmp_path / "magic.cgh")
    with pytest.raises(_lib.IoError):
        stages.read_cgh1(tmp_path / "absent.cgh")
    with pytest.raises(_lib.ValidationError):
        stages.read_cgh1(tmp_path / "nan.cgh")
    with pytest.raises(_lib.ValidationError):
        stages.write_cgh1(tmp_path / "x.cgh", plane, (0.0, 8e-6, 0.2))
