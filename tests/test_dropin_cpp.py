"""The reference's own C++ API backed by the GPU (integration/wavecgh_gpu.cpp
replacing synthesis.cpp, haar.cpp, saliency.cpp, angular_spectrum.cpp, fringe_lut.cpp) against
the unmodified CPU reference. The binary is built here by integration/Makefile (it needs the
reference headers) and travels to the GPU box prebuilt."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "integration" / "_build" / "dropin_check"


@pytest.mark.gpu
def test_reference_cpp_api_on_gpu_matches_reference():
    if not BIN.exists():
        pytest.skip("integration/_build not built (needs /root/reference at build time)")
    res = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(res.stdout[-3000:], res.stderr[-2000:])
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
    assert "PASSED" in res.stdout


def test_dropin_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available() or not BIN.exists():
        pytest.skip("needs the prebuilt binary and no GPU")
    res = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=120)
    assert res.returncode != 0
    assert "no CPU fallback" in res.stderr
