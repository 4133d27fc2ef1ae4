"""Row-band strong-scaling estimate on one GPU: each config's LAST band at
N = 1, 2, 4, 8 timed alone (CUDA events, warm, inputs resident).
  python tools/band_scaling.py > profiles/<tag>_band_scaling.jsonl"""
import sys, json, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2211_09938_b200 import _lib, scenes, tiles
from paper_2211_09938_b200.hologram import HologramJob, spec_for_scene
ctx = _lib.Context(0)
stream = torch.cuda.current_stream(); ctx.set_stream(stream.cuda_stream)
for cfg, method in ((1, "direct"), (2, "lut"), (3, "direct"), (4, "direct")):
    sc = scenes.make_scene(cfg)
    n = sc.config.plane_size
    obj = torch.from_numpy(sc.objects).cuda(); sal = torch.from_numpy(sc.masks).cuda()
    res = {}
    for world in (1, 2, 4, 8):
        r0, rows = tiles.band(world - 1, world, n)  # last rank's band
        job = HologramJob(spec_for_scene(sc, method=method, row0=r0, rows=rows), ctx)
        job.upload_dev(obj.data_ptr(), sal.data_ptr())
        job.run()
        reps = 3 if cfg < 3 else 1
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps): job.run()
        e1.record(stream); torch.cuda.synchronize()
        res[world] = e0.elapsed_time(e1) / reps
        job.close()
    eff = {w: res[1] / (w * res[w]) for w in res}
    print(json.dumps({"cfg": cfg, "method": method, "ms_band": res, "efficiency_est": eff}))
