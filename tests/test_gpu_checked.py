"""The checked build (libwcgh_checked.so, -DWCGH_CHECKED) in place of
compute-sanitizer, which is closed on this GPU pool
(profiles/r2_compute_sanitizer_closed.txt): device bounds checks on the LUT
windows (guarded allocations, wcgh_lut.cu), the shared weight array, the
partial planes, K3's point staging, K2's ballot-ranked compaction (record
count per segment == K1's count) and the fused gather's peer-plane stores;
scratch poisoned with 0xFF. Every C-ABI call collects the device flags.
Run in subprocesses (the library is chosen at load time by WCGH_CHECKED=1)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
CHECKED = ROOT / "paper_2211_09938_b200" / "libwcgh_checked.so"


def _run(code_or_args, env_extra=None, timeout=900):
    env = dict(os.environ, WCGH_CHECKED="1", **(env_extra or {}))
    args = code_or_args if isinstance(code_or_args, list) else [sys.executable, "-c", code_or_args]
    return subprocess.run(args, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


@pytest.fixture(scope="module", autouse=True)
def _need_checked_build():
    if not CHECKED.exists():
        pytest.fail("libwcgh_checked.so missing: run __graft_entry__.build()")


def test_checked_build_runs_the_sanitizer_cases_clean():
    """cfg0 through direct / LUT / FFT (+ fp64 phase, a row band), the u8
    front end at 48^2 and 144^2 (two layers), the device LUT / plane objects,
    reconstruction + SSIM, and the single-process multi-band path: no check
    fires, no poisoned value reaches a result."""
    r = _run([sys.executable, "tools/sanitize_cases.py"])
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count(": ok") == 5, r.stdout


def test_checked_build_catches_an_injected_compaction_fault():
    """Negative control: one extra count in K1's last segment makes K2's
    records disagree with the scan; the checked build reports it."""
    code = ("import sys; sys.path.insert(0, '.')\n"
            "from paper_2211_09938_b200 import scenes, _lib\n"
            "from paper_2211_09938_b200.hologram import HologramJob, spec_for_scene\n"
            "sc = scenes.make_scene(0)\n"
            "try:\n"
            "    HologramJob(spec_for_scene(sc))(sc.objects, sc.masks)\n"
            "    print('NO CHECK FIRED')\n"
            "except _lib.IoError as e:\n"
            "    print('caught:', e)\n")
    r = _run(code, {"WCGH_CHK_INJECT": "segcount"})
    assert r.returncode == 0, r.stderr
    assert "caught: checked build: device bounds check failed at wcgh_analysis.cu" in r.stdout, r.stdout
