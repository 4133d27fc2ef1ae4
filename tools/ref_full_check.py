"""Checks bench.py's extrapolated reference time at a 4096^2 config against
one FULL run of the reference's synthesize_progressive on the same host
(oracle/_ref, workers = nproc). Prints one JSON line: the two-window
extrapolation, the whole-hologram wall time, and their ratio."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2211_09938_b200 import scenes  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
estimate_only = "--estimate-only" in sys.argv
sc = scenes.make_scene(cfg)
t = bench.ReferenceTimer(sc)
try:
    t0 = time.perf_counter()
    est, desc = t.estimate(10.0)
    t_est = time.perf_counter() - t0
    t1 = time.perf_counter()
    full, fdesc = (float("nan"), "") if estimate_only else t.full()
    t_full = time.perf_counter() - t1
finally:
    t.close()
print(json.dumps({"config": sc.config.name, "extrapolated_s": est, "fit": t.fit,
                  "estimate_wall_s": t_est, "full_s": full, "full_wall_s": t_full,
                  "ratio_full_over_extrapolated": full / est, "workers": t.workers,
                  "nz_ops": t.nz_ops, "nz_by_stage": t.nz_by_stage, **bench.host_cpu()}))
