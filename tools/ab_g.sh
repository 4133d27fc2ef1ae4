#!/usr/bin/env bash
# K3 chirp: chunks per partial plane (default G vs G = 1), tests + cfg4/cfg1 timings
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-g}
mkdir -p "$OUT"
export WCGH_PARITY_LOG=$OUT/parity_$TAG.jsonl
rm -f $WCGH_PARITY_LOG
timeout 1500 python -m pytest tests -x -q -m gpu -k "direct or fixed or parity or band or tiles or peer or checked or multidepth or forms or full_plane" > "$OUT/tests_$TAG.log" 2>&1; echo "pytest=$?"; tail -2 "$OUT/tests_$TAG.log"
for g in def 1; do
  $( [ $g = def ] && echo "env -u WCGH_DIRECT_G" || echo "env WCGH_DIRECT_G=$g") timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > "$OUT/b4_${TAG}_G$g.json" 2>/dev/null; echo "b4 G=$g $?"
  $( [ $g = def ] && echo "env -u WCGH_DIRECT_G" || echo "env WCGH_DIRECT_G=$g") timeout 600 python bench.py --config 3 --steps 2 --warmup 2 --no-cpu-baseline --no-extra > "$OUT/b3_${TAG}_G$g.json" 2>/dev/null; echo "b3 G=$g $?"
done
