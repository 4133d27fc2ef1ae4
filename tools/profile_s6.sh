#!/usr/bin/env bash
# Session-6 GPU pass at HEAD (K3 with held run multipliers): smoke, the whole
# -m gpu suite, the driver's default bench line and reference arm, then the
# profiling set (every ncu run only after the identical plain command exited 0):
# launch list of the default bench (config 4), ncu --set full of one K3 launch at
# config 4 and at config 1, and the self-launched 2-rank bench on one device.
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-s6}
mkdir -p "$OUT"
export WCGH_PARITY_LOG=$OUT/parity_$TAG.jsonl
rm -f $WCGH_PARITY_LOG
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke_$TAG.log" 2>&1; echo "smoke=$?"
if [ -z "${SKIP_TESTS:-}" ]; then
timeout 1800 python -m pytest tests -x -q -m gpu --durations=15 > "$OUT/gputests_$TAG.log" 2>&1; echo "pytest=$?"; tail -n 2 "$OUT/gputests_$TAG.log"
fi
timeout 900 python bench.py > "$OUT/bench_$TAG.json" 2> "$OUT/bench_$TAG.err"; echo "bench=$?"
timeout 900 python bench.py --impl reference > "$OUT/bench_ref_$TAG.json" 2> "$OUT/bench_ref_$TAG.err"; echo "bench_ref=$?"
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
WCGH_BENCH_SAME_DEVICE=1 timeout 600 python bench.py --gpus 2 --config 1 --steps 5 --warmup 3 --no-cpu-baseline --no-extra \
  > "$OUT/bench_2rank_cfg1_$TAG.json" 2> "$OUT/bench_2rank_cfg1_$TAG.err"; echo "bench_2rank=$?"
