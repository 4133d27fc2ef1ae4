#!/usr/bin/env bash
# Profiling pass for one round (run on the GPU box through gpurun):
#   1. the default bench line (config 1, direct) with the CPU baseline;
#   2. ncu launch list of the same bench (device time of every launch);
#   3. ncu --set full of the top kernels: K1 analysis, K3 direct (config 1)
#      and K4 LUT stages (config 2).
# Every ncu command runs only after the identical plain command exited 0.
set -u
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r1}
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvsmi_$TAG.txt" 2>&1
timeout 600 python bench.py > "$OUT/bench_$TAG.json" 2> "$OUT/bench_$TAG.err"; echo "bench=$?"
B1="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
B2="python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline"
timeout 300 $B1 > "$OUT/plain1_$TAG.log" 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches_cfg1_$TAG.csv" $B1 > "$OUT/ncu1_$TAG.log" 2>&1; echo "ncu_launch=$?"
timeout 300 $B1 > "$OUT/plain2_$TAG.log" 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k "regex:k_analysis|k_direct_chirp" -s 2 -c 2 -o "$OUT/prof_k3_$TAG" $B1 > "$OUT/ncu2_$TAG.log" 2>&1; echo "ncu_k3=$?"
timeout 300 $B2 > "$OUT/plain3_$TAG.log" 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k "regex:k_lut_stage" -s 4 -c 4 -o "$OUT/prof_k4_$TAG" $B2 > "$OUT/ncu3_$TAG.log" 2>&1; echo "ncu_k4=$?"
