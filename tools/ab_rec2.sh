#!/usr/bin/env bash
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-ab}
mkdir -p "$OUT"
export WCGH_PARITY_LOG=$OUT/parity_$TAG.jsonl
rm -f $WCGH_PARITY_LOG
timeout 1200 python -m pytest tests -x -q -m gpu -k "direct or fixed or parity or band or tiles or peer or checked" > "$OUT/tests_$TAG.log" 2>&1; echo "pytest=$?"; tail -2 "$OUT/tests_$TAG.log"
for ru in 1 2; do
  WCGH_DIRECT_RU=$ru timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline --no-extra > "$OUT/b1_${TAG}_ru$ru.json" 2>/dev/null; echo "b1 ru=$ru $?"
  WCGH_DIRECT_RU=$ru timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra > "$OUT/b4_${TAG}_ru$ru.json" 2>/dev/null; echo "b4 ru=$ru $?"
done
