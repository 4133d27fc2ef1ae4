#!/usr/bin/env python
"""K1 + K2 (DWT, saliency pyramid, strict gates, A_eff, compaction) at large
object sizes on the GPU box: SURVEY.md §8(d) asks to prove the front end's
HBM bandwidth at >= 16384^2, where it is no longer launch-bound.

Algorithmic bytes per run: 1 B object + 1 B mask read and
4 B A_eff written per object pixel, plus 16 B per compacted point record.
Inputs are seeded synthetic uint8 objects (~30% nonzero) and 25%-salient
masks in 16 x 16-pixel blocks, generated on the device; the front end runs
through the C ABI's wcgh_job_analyze (no synthesis). One JSON line per size.

  python tools/bench_analysis.py [--sizes 2048,4096,8192,16384] [--reps 5]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_09938_b200 import _lib  # noqa: E402
from paper_2211_09938_b200.hologram import HologramJob, JobSpec  # noqa: E402


def inputs(n: int, seed: int):
    g = torch.Generator(device="cuda").manual_seed(seed)
    vals = torch.randint(1, 256, (n, n), generator=g, device="cuda", dtype=torch.int32)
    keep = torch.rand((n, n), generator=g, device="cuda") < 0.30
    obj = torch.where(keep, vals, torch.zeros_like(vals)).to(torch.uint8)
    blocks = (torch.rand((n // 16, n // 16), generator=g, device="cuda") < 0.25).to(torch.uint8)
    mask = (blocks.repeat_interleave(16, 0).repeat_interleave(16, 1) * 255).contiguous()
    return obj.contiguous(), mask


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="2048,4096,8192,16384")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    hbm = float(peaks["hbm_gbs"])
    ctx = _lib.Context(0)
    for n in (int(s) for s in args.sizes.split(",")):
        obj, mask = inputs(n, 1234 + n)
        job = HologramJob(JobSpec(object_size=n, plane_size=n, layers=[(532e-9, 8e-6, 0.2)],
                                  method="direct", rows=8), ctx)
        job.upload_dev(obj.data_ptr(), mask.data_ptr())
        job.analyze()  # warm-up
        ms = []
        st = None
        for _ in range(args.reps):
            st = job.analyze()
            ms.append(st["ms_analysis"])
        t = float(np.median(ms))
        pts = int(st["n_points"])
        algo = n * n * (1 + 1 + 4) + 16 * pts
        gbs = algo / (t * 1e-3) / 1e9
        print(json.dumps({
            "kernel": "K1+K2 front end (k_analysis, k_scan, k_compact_points)",
            "object": n, "points": pts, "ms": t,
            "algorithmic_bytes": algo, "achieved_gbs": gbs, "peak_gbs": hbm,
            "frac": gbs / hbm, "peak_basis": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)",
            "ops": st["ops"],
        }), flush=True)
        job.close()
        del obj, mask
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
