#!/usr/bin/env bash
# K4 variants at config 2 (LUT) and config 1: WCGH_LUT_DUFF=0/1/2, plus LUT parity tests per variant
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-k4}
mkdir -p "$OUT"
for v in ${VARIANTS:-0 1 2}; do
  WCGH_LUT_DUFF=$v timeout 600 python -m pytest tests -x -q -m gpu -k "lut" > "$OUT/tests_${TAG}_d$v.log" 2>&1; echo "tests d=$v $? $(tail -1 $OUT/tests_${TAG}_d$v.log)"
  WCGH_LUT_DUFF=$v timeout 600 python bench.py --config 2 --method lut --steps 5 --warmup 2 --no-cpu-baseline --no-extra > "$OUT/b2_${TAG}_d$v.json" 2>/dev/null; echo "b2 d=$v $?"
done
