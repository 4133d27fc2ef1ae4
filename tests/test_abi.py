"""The C-ABI library loads and exports every symbol include/wcgh.h declares;
without a GPU it fails loudly (no CPU fallback)."""
import ctypes
import re

import pytest

from conftest import ROOT
from paper_2211_09938_b200 import _lib


def header_symbols():
    text = (ROOT / "include" / "wcgh.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(wcgh_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTED) == declared
    assert lib.wcgh_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_lib.Point) == 16
    assert ctypes.sizeof(_lib.Layer) == 24
    assert ctypes.sizeof(_lib.Plan) == 40


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.IoError, match="no CUDA device"):
        _lib.Context(0)
