#!/usr/bin/env python
"""K3 held run multipliers (WCGH_DIRECT_HOLD = 1, 2, 4): error against the fp64
Eq.(1) oracle on the BASELINE geometries (random points over the object area,
plane rows incl. the corners), relative L2 and the worst pixel. Run on the GPU box:
    python tools/hold_error.py > gpurun_out/hold_error.jsonl
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import oracle as O  # noqa: E402  (checker only)
from paper_2211_09938_b200 import _lib, stages  # noqa: E402

WL = 532e-9
GEOMS = {  # name: plane, layers, object half-width
    "cfg1_1024_p8_z0.20": (1024, [(WL, 8e-6, 0.2)], 256),
    "cfg2_2048_p8_z0.20": (2048, [(WL, 8e-6, 0.2)], 512),
    "cfg3_4096_p4_z0.15-0.30": (4096, [(WL, 4e-6, z) for z in (0.15, 0.20, 0.25, 0.30)], 512),
    "cfg4_4096_p4_z0.20": (4096, [(WL, 4e-6, 0.2)], 1024),
}


def main():
    for name, (nh, layers, half) in GEOMS.items():
        rng = np.random.default_rng(99)
        n = 3000
        pts = np.zeros(n, _lib.POINT_DTYPE)
        pts["x"] = rng.integers(nh // 2 - half, nh // 2 + half, n)
        pts["y"] = rng.integers(nh // 2 - half, nh // 2 + half, n)
        pts["a"] = rng.integers(1, 256, n).astype(np.float32)
        pts["layer"] = np.sort(rng.integers(0, len(layers), n))
        rows = (0, nh // 4, nh // 2, nh - 1)
        py, px = np.meshgrid(np.asarray(rows), np.arange(nh), indexing="ij")
        ref = O.direct_pixels(pts["x"], pts["y"], pts["a"], pts["layer"], layers, px.ravel(),
                              py.ravel()).reshape(len(rows), nh)
        for hold in ("auto", "1", "2", "4"):
            if hold == "auto":
                os.environ.pop("WCGH_DIRECT_HOLD", None)
            else:
                os.environ["WCGH_DIRECT_HOLD"] = hold
            got = np.stack([stages.synth_points(pts, layers, nh, row0=r, rows=1)[0] for r in rows])
            d = np.abs(got - ref)
            print(json.dumps({
                "geometry": name, "hold": hold, "rel_l2": O.rel_l2(got, ref),
                "rel_l2_corner_row": O.rel_l2(got[0], ref[0]),
                "worst_pixel_abs_over_rms": float(d.max() / np.sqrt(np.mean(np.abs(ref) ** 2))),
            }), flush=True)


if __name__ == "__main__":
    main()
