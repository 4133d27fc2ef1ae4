"""In-tree build of libwcgh.so (sm_100a) with nvcc.

The shared library lands next to this file so it travels with the repo
snapshot to the GPU box; no JIT cache is involved.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "wcgh"
LIB = PKG / "libwcgh.so"
SOURCES = ["wcgh_analysis.cu", "wcgh_direct.cu", "wcgh_lut.cu", "wcgh_fft.cu", "wcgh_recon.cu",
           "wcgh_abi.cu", "wcgh_job.cu", "wcgh_io.cu", "wcgh_lutobj.cu", "wcgh_helpers.cu", "wcgh_fftk.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]


def _run(cmd: list[str], log: Path | None = None) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd)}")


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> Path:
    """libwcgh.so (the product), or with checked=True libwcgh_checked.so: the
    same sources with -DWCGH_CHECKED (device bounds checks, poisoned scratch;
    test use only, loaded when WCGH_CHECKED=1). Translation units compile in
    parallel."""
    from concurrent.futures import ThreadPoolExecutor

    out_dir = BUILD.parent / ("wcgh_checked" if checked else "wcgh")
    lib = PKG / ("libwcgh_checked.so" if checked else "libwcgh.so")
    out_dir.mkdir(parents=True, exist_ok=True)
    deps = [CSRC / s for s in SOURCES] + [CSRC / "wcgh_internal.cuh", CSRC / "wcgh_state.cuh",
                                           ROOT / "include" / "wcgh.h"]
    newest = max(p.stat().st_mtime for p in deps)
    if lib.exists() and lib.stat().st_mtime >= newest and not force:
        return lib
    extra = ["-DWCGH_CHECKED"] if checked else []
    # tuning builds only, e.g. WCGH_NVCC_EXTRA=-DWCGH_LUT_SWEEP (more K4 window shapes)
    extra += os.environ.get("WCGH_NVCC_EXTRA", "").split()

    def one(src):
        obj = out_dir / (Path(src).stem + ".o")
        _run([NVCC, *ARCH, *FLAGS, *extra, "-c", str(CSRC / src), "-o", str(obj)],
             log=out_dir / (Path(src).stem + ".ptxas.log"))
        return str(obj)

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(one, SOURCES))
    if verbose:
        for src in SOURCES:
            print((out_dir / (Path(src).stem + ".ptxas.log")).read_text())
    tmp = lib.with_suffix(".so.tmp")
    _run([NVCC, *ARCH, "-shared", "-o", str(tmp), *objs, "-lcudart_static", "-lrt", "-ldl",
          "-lpthread", "-Xlinker", "-rpath=/usr/local/cuda/lib64"])
    tmp.replace(lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    if "--checked" in sys.argv:
        print(build(force="--force" in sys.argv, checked=True))
