#!/usr/bin/env bash
# K4 run-gap threshold x chunk target sweep at config 2 (LUT), kernel times
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-gap}
mkdir -p "$OUT"
for ch in ${CHUNKS:-4 8 16}; do for g in ${GAPS:-2 4 8}; do
  WCGH_LUT_GAP=$g WCGH_LUT_CHUNKS=$ch timeout 300 python bench.py --config 2 --method lut --steps 5 --warmup 2 --no-cpu-baseline --no-extra > "$OUT/b2_${TAG}_g${g}_c${ch}.json" 2>/dev/null
  python -c "
import json;d=json.loads(open('$OUT/b2_${TAG}_g${g}_c${ch}.json').read().strip().splitlines()[-1]);r=d['roofline']
print('gap $g chunks $ch','ms',round(d['ms_per_step'],3),'kernel_ms',round(r.get('kernel_ms',0),3),'frac',round(r['frac'],4))"
done; done
