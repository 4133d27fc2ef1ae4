#!/usr/bin/env python
"""Real vs random-initial-phase (complex) objects on BASELINE.json's
configuration 1 geometry, through each synthesis method (GPU box).

The complex object is the reference's random_phase_field of the config's
object (amplitude = u8 / 255, seed 424242; synthesis.cpp:205-214, drawn on
the host by wcgh_random_phase_field) with the config's mask as saliency; the
real run uses the same amplitude as an f64 object. One JSON line per
(method, object kind): device ms per hologram (CUDA events on the job
stream, warm, median), points / cells, and the synthesis-kernel time.

  python tools/bench_complex.py [--steps 5] > profiles/rN_complex.jsonl
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

from paper_2211_09938_b200 import _lib, scenes, stages  # noqa: E402
from paper_2211_09938_b200.hologram import HologramJob, spec_for_scene  # noqa: E402


def timed(job, obj, sal, steps, stream):
    job.upload_dev(obj.data_ptr(), sal.data_ptr())
    job.run()  # warm-up
    ms = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        job.run()
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return float(np.median(ms)), job.stats()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    sc = scenes.make_scene(args.config)
    amp = sc.objects[0].astype(np.float64) / 255.0
    rot = stages.random_phase_field(amp, 424242)
    sal = torch.from_numpy(sc.masks[0].astype(np.float64) / 255.0).cuda()
    inputs = {"real": ("f64", torch.from_numpy(amp).cuda()),
              "complex": ("c128", torch.from_numpy(rot).cuda())}
    ctx = _lib.Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    for method in ("direct", "lut", "fft"):
        for kind, (dt, obj) in inputs.items():
            spec = spec_for_scene(sc, method=method)
            spec.obj_dtype, spec.sal_dtype, spec.obj_scale = dt, "f64", 1.0
            job = HologramJob(spec, ctx)
            ms, st = timed(job, obj, sal, args.steps, stream)
            job.close()
            print(json.dumps({"config": args.config, "method": method, "object": kind,
                              "ms": ms, "ms_synthesis": st["ms_synthesis"],
                              "ms_analysis": st["ms_analysis"], "n_points": st["n_points"],
                              "updates": st["updates"],
                              "synth_launches": st["synth_launches"]}), flush=True)


if __name__ == "__main__":
    main()
