#!/usr/bin/env bash
# ncu --set full (+source) of K4's B=1 stage at config 2 (after the plain run exited 0)
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-k4p}
mkdir -p "$OUT"
B2="python bench.py --config 2 --method lut --steps 1 --warmup 1 --no-cpu-baseline --no-extra"
timeout 300 $B2 > "$OUT/plain2_$TAG.log" 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on \
    -k "regex:k_lut_stage" -s 3 -c 1 -o "$OUT/prof_k4b1_$TAG" $B2 > "$OUT/ncu_k4b1_$TAG.log" 2>&1; echo "ncu=$?"
