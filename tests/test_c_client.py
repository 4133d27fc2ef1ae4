"""The C ABI from plain C (examples/synth_c.c, what a cgo/JNI/ctypes binding
does): the header compiles as strict C99, the client fails loudly without a
GPU and, on the B200, synthesises with all three methods, round-trips CGH1
and reconstructs + scores through the ABI."""
import subprocess
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_2211_09938_b200"


def _build(tmp_path):
    exe = tmp_path / "synth_c"
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-pedantic", "-Werror",
           f"-I{ROOT / 'include'}", str(ROOT / "examples" / "synth_c.c"), f"-L{LIBDIR}",
           "-l:libwcgh.so", f"-Wl,-rpath,{LIBDIR}", "-lm", "-o", str(exe)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return exe


def test_header_is_c99_and_client_fails_loudly_without_gpu(tmp_path):
    if not (LIBDIR / "libwcgh.so").exists():
        pytest.skip("libwcgh.so not built")
    exe = _build(tmp_path)
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu test")
    res = subprocess.run([str(exe), str(tmp_path / "x.cgh")], capture_output=True, text=True)
    assert res.returncode == 2 and "no CPU fallback" in res.stderr


@pytest.mark.gpu
def test_c_client_on_gpu(tmp_path):
    exe = _build(tmp_path)
    res = subprocess.run([str(exe), str(tmp_path / "x.cgh")], capture_output=True, text=True,
                         timeout=300)
    print(res.stdout, res.stderr)
    assert res.returncode == 0 and "PASSED" in res.stdout, res.stdout + res.stderr
