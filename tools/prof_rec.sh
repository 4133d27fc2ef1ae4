#!/usr/bin/env bash
# K3 recurrence form: point-loop unroll A/B at configs 1 and 4, then one
# `ncu --set full` capture of a config-1 K3 launch (after the plain run exited 0).
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-rec}
mkdir -p "$OUT"
for ru in 1 2; do
  WCGH_DIRECT_RU=$ru timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline --no-extra > "$OUT/b1_${TAG}_ru$ru.json" 2>/dev/null; echo "b1 ru=$ru $?"
  WCGH_DIRECT_RU=$ru timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra > "$OUT/b4_${TAG}_ru$ru.json" 2>/dev/null; echo "b4 ru=$ru $?"
done
B1="python bench.py --config 1 --steps 1 --warmup 1 --no-cpu-baseline --no-extra"
timeout 300 $B1 > "$OUT/plain1_$TAG.log" 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on \
    -k "regex:k_direct_rec" -s 1 -c 1 -o "$OUT/prof_k3rec_cfg1_$TAG" $B1 > "$OUT/ncu_k3rec_$TAG.log" 2>&1; echo "ncu=$?"
