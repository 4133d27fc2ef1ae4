import sys, time
sys.path.insert(0, '.')
import torch
from paper_2211_09938_b200 import _lib, scenes
from paper_2211_09938_b200.hologram import HologramJob, spec_for_scene
ctx = _lib.Context(0)
sc = scenes.make_scene(2)
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    job = HologramJob(spec_for_scene(sc, method="lut"), ctx)
    torch.cuda.synchronize(); print("job create ms", (time.perf_counter() - t) * 1e3)
    job.close()
