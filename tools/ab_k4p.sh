#!/usr/bin/env bash
# K4 A/B: run-list chunks as kernel parameter blocks (WCGH_LUT_PARAMS=1, uniform-register
# weights) vs the shared-memory form (0): LUT tests, then config-2 / config-1 LUT kernel time.
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-k4p}
mkdir -p "$OUT"
timeout 900 python -m pytest tests -x -q -m gpu -k "lut or cfg2 or LUT" > "$OUT/tests_${TAG}.log" 2>&1; echo "tests $? $(tail -1 $OUT/tests_${TAG}.log)"
for p in ${MODES:-1 0}; do
  for cfg in 2 1; do
    WCGH_LUT_PARAMS=$p timeout 600 python bench.py --config $cfg --method lut --steps 5 --warmup 3 --no-cpu-baseline --no-extra > "$OUT/b${cfg}_${TAG}_p$p.json" 2> "$OUT/b${cfg}_${TAG}_p$p.err"
    python -c "
import json,sys
d=json.loads(open('$OUT/b${cfg}_${TAG}_p$p.json').read().strip().splitlines()[-1]); r=d['roofline']
print('params=$p cfg$cfg: %.3f ms/holo  kernel %.3f ms  frac %.4f' % (d['ms_per_step'], r['kernel_ms'], r['frac']))" 2>&1 | tail -1
  done
done
