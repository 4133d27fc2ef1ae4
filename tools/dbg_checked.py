import sys, numpy as np
sys.path.insert(0, ".")
from paper_2211_09938_b200 import scenes, stages, _lib
from paper_2211_09938_b200.hologram import HologramJob, spec_for_scene
print("lib", _lib.LIB_PATH.name)
for cfg in (0, 1):
    sc = scenes.make_scene(cfg)
    for m in ("direct", "lut", "fft"):
        j = HologramJob(spec_for_scene(sc, method=m))
        h = j(sc.objects, sc.masks)
        st = j.stats()
        print(cfg, m, "norm", float(np.linalg.norm(h)), "nan", int(np.isnan(h).sum()), "pts", st["n_points"], "launches", st["total_launches"])
pts = np.zeros(3, _lib.POINT_DTYPE); pts["x"] = [10, 500, 900]; pts["y"] = [10, 500, 900]; pts["a"] = 1
for nh in (128, 512, 1024):
    r = stages.synth_points(pts[pts["x"] < nh], [(532e-9, 8e-6, 0.2)], nh)
    print("synth_points", nh, float(np.abs(r).sum()))
