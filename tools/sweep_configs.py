#!/usr/bin/env python
"""All BASELINE.json configs through the three synthesis methods (GPU box).

Prints one JSON line per (config, saliency fraction, method): device
ms/hologram (CUDA events on the job stream, warm), P or nonzero-cell count,
updates/s with the config's numerator (P * Nh^2 for direct configs, nonzero
cells * Nh^2 for the LUT config), and the kernel time split.

  python tools/sweep_configs.py [--quick] > profiles/rN_configs.jsonl
  python tools/sweep_configs.py --md profiles/rN_configs.jsonl > profiles/rN_configs.md
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_09938_b200 import _lib, scenes  # noqa: E402
from paper_2211_09938_b200.hologram import HologramJob, spec_for_scene  # noqa: E402


def run(sc, method, steps, ctx):
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    t0 = time.perf_counter()
    job = HologramJob(spec_for_scene(sc, method=method), ctx)
    setup_s = time.perf_counter() - t0
    obj = torch.from_numpy(sc.objects).cuda()
    sal = torch.from_numpy(sc.masks).cuda()
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
    st = job.stats()
    job.close()
    return float(np.median(ms)), st, setup_s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--md", default=None, help="render a jsonl produced by this tool as markdown")
    args = ap.parse_args()
    if args.md:
        render_md(args.md)
        return
    ctx = _lib.Context(0)
    cases = [(0, None), (1, None), (2, None), (3, None)]
    cases += [(4, f) for f in (0.0, 0.10, 0.25, 0.50, 1.0)]
    if args.quick:
        cases = [(0, None), (1, None), (2, None)]
    for cfg, frac in cases:
        sc = scenes.make_scene(cfg, saliency_frac=frac)
        c = sc.config
        res = {}
        for method in ("direct", "lut", "fft"):
            big = c.plane_size >= 4096 and method == "direct"
            res[method] = run(sc, method, 1 if big else 3, ctx)
        points = res["direct"][1]["n_points"]
        cells = res["lut"][1]["n_points"]
        numer = (cells if c.method == "lut" else points) * c.plane_size ** 2
        for method, (ms, st, setup) in res.items():
            print(json.dumps({
                "config": c.name, "saliency_frac": c.saliency_frac, "method": method,
                "ms_per_hologram": ms, "points": points, "lut_cells": cells,
                "numerator": "nonzero cells x Nh^2" if c.method == "lut" else "points x Nh^2",
                "updates_per_s": numer / (ms * 1e-3),
                "kernel_updates_per_s": st["updates"] / (st["ms_synthesis"] * 1e-3) if st["ms_synthesis"] else None,
                "ms_analysis": st["ms_analysis"], "ms_synthesis": st["ms_synthesis"],
                "ms_reduce": st["ms_reduce"], "ops": st["ops"], "setup_s": setup,
            }), flush=True)


def render_md(path):
    rows = [json.loads(line) for line in open(path) if line.strip().startswith("{")]
    print("# All configs, three synthesis methods (B200, device time per hologram, warm)\n")
    print("Command: `python tools/sweep_configs.py` (one job per row; inputs resident in HBM; "
          "CUDA events). `updates/s` uses the config's numerator (points x Nh^2 for direct "
          "configs, nonzero gated cells x Nh^2 for config 2); `kernel upd/s` is the synthesis "
          "kernel's own algorithmic rate (points x pixels for direct, nonzero cells x pixels for "
          "LUT; none for FFT).\n")
    print("| config | saliency | method | ms/hologram | points P | LUT cells | updates/s | kernel upd/s |")
    print("|---|---|---|---|---|---|---|---|")
    for r in rows:
        k = r.get("kernel_updates_per_s")
        print(f"| {r['config']} | {r['saliency_frac']:.2f} | {r['method']} | {r['ms_per_hologram']:.2f} "
              f"| {r['points']} | {r['lut_cells']} | {r['updates_per_s']:.3g} | "
              f"{'%.3g' % k if k else '-'} |")


if __name__ == "__main__":
    main()
