#!/usr/bin/env bash
# compute-sanitizer pass: memcheck, racecheck, synccheck
# and initcheck over tools/sanitize_cases.py, plus memcheck over the
# two-process fused peer gather. Summaries -> $OUT/sanitize_*.txt
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 python tools/sanitize_cases.py \
    > "$OUT/sanitize_$tool.txt" 2>&1
  echo "$tool rc=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' "$OUT/sanitize_$tool.txt" | tr '\n' ' ')"
done
timeout 900 $CS --tool memcheck --target-processes all --print-limit 50 \
  python -m pytest tests/test_gpu_peer_gather.py -x -q -k direct > "$OUT/sanitize_peer_gather.txt" 2>&1
echo "peer_gather memcheck rc=$?: $(grep -E 'ERROR SUMMARY|passed|failed' "$OUT/sanitize_peer_gather.txt" | tr '\n' ' ')"
