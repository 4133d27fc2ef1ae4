#!/usr/bin/env bash
# K4 A/B: the run-by-run kernel (WCGH_LUT_KERNEL=runs) vs the stream kernel,
# bitwise-equal planes, then kernel time at configs 2 and 1 (LUT method).
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
cat > /tmp/k4_dump.py <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2211_09938_b200 import scenes
from paper_2211_09938_b200.hologram import HologramJob, spec_for_scene
out = {}
for cfg in (1, 2):
    sc = scenes.make_scene(cfg)
    j = HologramJob(spec_for_scene(sc, method="lut"))
    out[f"cfg{cfg}"] = j(sc.objects, sc.masks)
np.savez(sys.argv[1], **out)
PY
WCGH_LUT_KERNEL=runs python /tmp/k4_dump.py /tmp/k4_runs.npz && python /tmp/k4_dump.py /tmp/k4_stream.npz && \
python -c "
import numpy as np
a=np.load('/tmp/k4_runs.npz'); b=np.load('/tmp/k4_stream.npz')
for k in a.files: print(k, 'bitwise equal' if np.array_equal(a[k], b[k]) else 'DIFFERENT')
"
for kern in ${KERNELS:-runs stream}; do
  for cfg in 2 1; do
    r=$(WCGH_LUT_KERNEL=$kern timeout 300 python bench.py --config $cfg --method lut --steps 5 --warmup 2 --no-cpu-baseline --no-extra 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('%.3f ms/holo  kernel %.3f ms  frac %.4f' % (d['ms_per_step'], r['kernel_ms'], r['frac']))" 2>&1)
    echo "kernel=$kern cfg$cfg lut: $r"
  done
done
