import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2211_09938_b200 import scenes
from paper_2211_09938_b200.hologram import HologramJob, spec_for_scene
sc = scenes.make_scene(0)
job = HologramJob(spec_for_scene(sc, method="fft"))
h = job(sc.objects, sc.masks)
print("ok", np.abs(h).max())
