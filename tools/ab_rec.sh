#!/usr/bin/env bash
# A/B of the direct kernel forms: per-pixel (WCGH_DIRECT_REC=0) vs the
# angle-addition recurrence (default): parity of every direct test, then
# cfg4 / cfg1 bench lines of each.
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-ab}
mkdir -p "$OUT"
export WCGH_PARITY_LOG=$OUT/parity_$TAG.jsonl
rm -f $WCGH_PARITY_LOG
timeout 1200 python -m pytest tests -x -q -m gpu -k "direct or fixed or parity or band or tiles or peer or checked" > "$OUT/tests_$TAG.log" 2>&1; echo "pytest=$?"; tail -2 "$OUT/tests_$TAG.log"
for rec in 1 0; do
  WCGH_DIRECT_REC=$rec timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > "$OUT/b4_${TAG}_rec$rec.json" 2> "$OUT/b4_${TAG}_rec$rec.err"; echo "b4 rec=$rec $?"
  WCGH_DIRECT_REC=$rec timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline --no-extra > "$OUT/b1_${TAG}_rec$rec.json" 2> "$OUT/b1_${TAG}_rec$rec.err"; echo "b1 rec=$rec $?"
done
