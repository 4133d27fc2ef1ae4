#!/usr/bin/env bash
# direct kernel forms: 2 = chirp-factored recurrence (default), 1 = sigma recurrence, 0 = per-pixel
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-ab}
mkdir -p "$OUT"
export WCGH_PARITY_LOG=$OUT/parity_$TAG.jsonl
rm -f $WCGH_PARITY_LOG
timeout 1200 python -m pytest tests -x -q -m gpu -k "direct or fixed or parity or band or tiles or peer or checked or multidepth" > "$OUT/tests_$TAG.log" 2>&1; echo "pytest=$?"; tail -2 "$OUT/tests_$TAG.log"
for rec in ${RECS:-2 1}; do
  WCGH_DIRECT_REC=$rec timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline --no-extra > "$OUT/b1_${TAG}_rec$rec.json" 2>/dev/null; echo "b1 rec=$rec $?"
  WCGH_DIRECT_REC=$rec timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra > "$OUT/b4_${TAG}_rec$rec.json" 2>/dev/null; echo "b4 rec=$rec $?"
done
WCGH_DIRECT_REC=2 timeout 600 python bench.py --config 3 --steps 1 --warmup 2 --no-cpu-baseline --no-extra > "$OUT/b3_${TAG}_rec2.json" 2>/dev/null; echo "b3 $?"
