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


# ---- CGHL LUT cache files (fringe_lut.cpp:95-166) ------------------------------

def test_cghl_bytes_identical_to_reference_writer(tmp_path):
    """Our writer, given the reference's LUT samples, produces the reference's
    own CGHL file byte for byte (header + f32 payload, lut_cache_store)."""
    from conftest import golden
    g = golden("ref_cghl_n16_b2")
    p = tmp_path / "lut.cghl"
    stages.write_cghl(p, g["lut"].astype(np.complex64), 16, 2, (532e-9, 8e-6, 0.1))
    assert p.read_bytes() == g["cghl_bytes"].tobytes()
    # and reads the reference's file back (lut_cache_load's header fields)
    ref_file = tmp_path / "ref.cghl"
    ref_file.write_bytes(g["cghl_bytes"].tobytes())
    lut, n, block, scene = stages.read_cghl(ref_file)
    assert (n, block, scene) == (16, 2, (532e-9, 8e-6, 0.1))
    assert np.array_equal(lut, g["lut"].astype(np.complex64))
    magic, version, b, size = struct.unpack("<4sHHI", g["cghl_bytes"].tobytes()[:12])
    assert (magic, version, b, size) == (b"CGHL", 1, 2, 16)


def test_cghl_errors(tmp_path):
    from conftest import golden
    raw = golden("ref_cghl_n16_b2")["cghl_bytes"].tobytes()
    cases = {"magic": b"XGHL" + raw[4:], "version": raw[:4] + b"\x02\x00" + raw[6:],
             "truncated": raw[:-8], "header": raw[:20]}
    for name, data in cases.items():
        p = tmp_path / f"{name}.cghl"
        p.write_bytes(data)
        with pytest.raises(_lib.IoError):
            stages.read_cghl(p)
    with pytest.raises(_lib.IoError):
        stages.read_cghl(tmp_path / "missing.cghl")
    with pytest.raises(_lib.ValidationError):
        stages.write_cghl(tmp_path / "x.cghl", np.zeros((5, 5), np.complex64), 16, 2, (532e-9, 8e-6, 0.1))
