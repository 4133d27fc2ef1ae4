#!/usr/bin/env bash
# Round-2 profiling pass (one GPU; every ncu run only after the identical
# plain command exited 0):
#   1. launch list of the default bench (config 4, direct)  -> launches_cfg4
#   2. ncu --set full of one K3 launch at config 4          -> prof_k3_cfg4
#   3. ncu --set full of the four K4 stages at config 2     -> prof_k4_cfg2
set -u
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r2}
mkdir -p "$OUT"
B4="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extra"
B2="python bench.py --config 2 --method lut --steps 1 --warmup 1 --no-cpu-baseline --no-extra"
if [ -z "${SKIP_LAUNCHES:-}" ]; then
timeout 900 $B4 > "$OUT/plain4_$TAG.log" 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches_cfg4_$TAG.csv" $B4 > "$OUT/ncu_l4_$TAG.log" 2>&1; echo "ncu_launch=$?"
fi
if [ -z "${SKIP_K3:-}" ]; then
timeout 900 $B4 > "$OUT/plain4b_$TAG.log" 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on \
    -k "regex:k_direct_chirp" -s 2 -c 1 -o "$OUT/prof_k3_cfg4_$TAG" $B4 > "$OUT/ncu_k3_$TAG.log" 2>&1; echo "ncu_k3=$?"
fi
if [ -z "${SKIP_K4:-}" ]; then
timeout 300 $B2 > "$OUT/plain2_$TAG.log" 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on \
    -k "regex:k_lut_st" -s 4 -c 4 -o "$OUT/prof_k4_cfg2_$TAG" $B2 > "$OUT/ncu_k4_$TAG.log" 2>&1; echo "ncu_k4=$?"
fi
