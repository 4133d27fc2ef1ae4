#!/usr/bin/env bash
# Session-3 GPU pass: whole -m gpu suite, then the profiling set for the new
# K3 (every ncu run only after the identical plain command exited 0):
#   launch list of the default bench (config 4), ncu --set full of one K3
#   launch at config 4 and at config 1.
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-s3}
mkdir -p "$OUT"
export WCGH_PARITY_LOG=$OUT/parity_$TAG.jsonl
rm -f $WCGH_PARITY_LOG
if [ -z "${SKIP_TESTS:-}" ]; then
timeout 1800 python -m pytest tests -x -q -m gpu > "$OUT/gputests_$TAG.log" 2>&1; echo "pytest=$?"; tail -2 "$OUT/gputests_$TAG.log"
fi
B4="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extra"
B1="python bench.py --config 1 --steps 1 --warmup 1 --no-cpu-baseline --no-extra"
timeout 900 $B4 > "$OUT/plain4_$TAG.log" 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches_cfg4_$TAG.csv" $B4 > "$OUT/ncu_l4_$TAG.log" 2>&1; echo "ncu_launch=$?"
timeout 900 $B4 > "$OUT/plain4b_$TAG.log" 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on \
    -k "regex:k_direct_chirp" -s 2 -c 1 -o "$OUT/prof_k3_cfg4_$TAG" $B4 > "$OUT/ncu_k3_$TAG.log" 2>&1; echo "ncu_k3_4=$?"
timeout 300 $B1 > "$OUT/plain1_$TAG.log" 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on \
    -k "regex:k_direct_chirp" -s 1 -c 1 -o "$OUT/prof_k3_cfg1_$TAG" $B1 > "$OUT/ncu_k3_1_$TAG.log" 2>&1; echo "ncu_k3_1=$?"
