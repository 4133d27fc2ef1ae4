"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): config 0 through every synthesis method, the uint8 front end at
odd sizes (partial 128-px segments), the device LUT / plane objects, the
reconstruction + SSIM kernels and the single-process multi-band path.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2211_09938_b200 import _lib, scenes, stages  # noqa: E402
from paper_2211_09938_b200.hologram import HologramJob, JobSpec, spec_for_scene, synthesize_multi  # noqa: E402

WL = 532e-9


def cfg0_methods():
    sc = scenes.make_scene(0)
    for method in ("direct", "lut", "fft"):
        job = HologramJob(spec_for_scene(sc, method=method))
        h = job(sc.objects, sc.masks)
        job.download_stages()
        assert np.isfinite(h).all()
        job.close()
    # fp64 phase mode and a row band
    job = HologramJob(spec_for_scene(sc, phase="fp64", row0=17, rows=40))
    job(sc.objects, sc.masks)
    job.close()


def front_end_odd():
    rng = np.random.default_rng(11)
    for n in (48, 144):
        objs = rng.integers(0, 256, (2, n, n), dtype=np.uint8)
        masks = rng.integers(0, 256, (2, n, n), dtype=np.uint8)
        plane = 64
        while plane < n or (plane - n) % 16:
            plane *= 2
        job = HologramJob(JobSpec(object_size=n, plane_size=plane,
                                  layers=[(WL, 8e-6, 0.2), (WL, 8e-6, 0.21)], rows=8))
        job.upload(objs, masks)
        job.analyze()
        job.download_a_eff()
        job.download_points()
        job.close()
        stages.analyze(objs[0].astype(np.float64), masks[0] / 255.0)


def lut_objects():
    n = 32
    lay = (WL, 8e-6, 0.1)
    rng = np.random.default_rng(2)
    plane = stages.DevicePlane(n)
    for b in (1, 2, 4, 8):
        lut = stages.DeviceLut(lay, n, b)
        m = n // b
        cells = rng.integers(0, m * m, 20)
        lut.apply_blocks(plane, cells, rng.random(20), rng.random(20))
    h, v, d = rng.standard_normal((3, n // 4, n // 4))
    stages.DeviceLut(lay, n, 2).refine(plane, h, v, d, rng.random((n // 2, n // 2)), 0.5)
    plane.download(np.complex128)


def recon_ssim():
    sc = scenes.make_scene(0)
    job = HologramJob(spec_for_scene(sc))
    holo = job(sc.objects, sc.masks)
    r = stages.reconstruct(holo, (WL, 8e-6, 0.2))
    stages.ssim(r, r * 1.01, 8, 0.01, 0.03, float(r.max() - r.min()))
    job.reconstruct()
    job.close()


def multi_band():
    sc = scenes.make_scene(0)
    for method in ("direct", "lut", "fft"):
        synthesize_multi(spec_for_scene(sc, method=method), sc.objects, sc.masks, [0, 0])


CASES = {"cfg0_methods": cfg0_methods, "front_end_odd": front_end_odd, "lut_objects": lut_objects,
         "recon_ssim": recon_ssim, "multi_band": multi_band}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    _lib.default_context()
    for name in names:
        CASES[name]()
        print(f"case {name}: ok", flush=True)
