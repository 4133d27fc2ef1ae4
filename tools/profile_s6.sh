#!/usr/bin/env bash
# Session-6 GPU pass at HEAD (K3 with held run multipliers, v_0 seeded at the first
# sub-run's middle): smoke, the whole -m gpu suite, the hold error tool, the driver's
# default bench line and reference arm, the self-launched 2-rank bench on one device
# (functional), then the profiling set (every ncu run only after the identical plain
# command exited 0): launch list of the default bench (config 4), ncu --set full of one
# K3 launch at config 4 and at config 1. The .ncu-rep files are summarised on the box
# (tools/ncu_summary.py + the raw and source pages as csv) and only kept while
# gpurun_out stays under the 64 MiB that travels back.
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-s6}
mkdir -p "$OUT"
export WCGH_PARITY_LOG=$OUT/parity_$TAG.jsonl
rm -f $WCGH_PARITY_LOG
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke_$TAG.log" 2>&1; echo "smoke=$?"
if [ -z "${SKIP_TESTS:-}" ]; then
timeout 1800 python -m pytest tests -x -q -m gpu --durations=15 > "$OUT/gputests_$TAG.log" 2>&1; echo "pytest=$?"; tail -n 2 "$OUT/gputests_$TAG.log"
fi
python tools/hold_error.py > $OUT/hold_error_$TAG.jsonl 2> $OUT/hold_error_$TAG.err; echo hold_err=$?
timeout 900 python bench.py > "$OUT/bench_$TAG.json" 2> "$OUT/bench_$TAG.err"; echo "bench=$?"
timeout 900 python bench.py --impl reference > "$OUT/bench_ref_$TAG.json" 2> "$OUT/bench_ref_$TAG.err"; echo "bench_ref=$?"
WCGH_BENCH_SAME_DEVICE=1 WCGH_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --config 1 --steps 5 --warmup 3 --no-cpu-baseline --no-extra \
  > "$OUT/bench_2rank_cfg1_$TAG.json" 2> "$OUT/bench_2rank_cfg1_$TAG.err"; echo "bench_2rank=$?"
B4="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extra"
B1="python bench.py --config 1 --steps 1 --warmup 1 --no-cpu-baseline --no-extra"
timeout 900 $B4 > "$OUT/plain4_$TAG.log" 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches_cfg4_$TAG.csv" $B4 > "$OUT/ncu_l4_$TAG.log" 2>&1; echo "ncu_launch=$?"
summarise() {  # $1 = report stem, $2 = md name
  if [ -f "$1.ncu-rep" ]; then
    python tools/ncu_summary.py report "$1.ncu-rep" > "$OUT/$2.md" 2> "$OUT/$2.err"
    python tools/ncu_summary.py traffic "$1.ncu-rep" > "$OUT/$2.traffic.json" 2>> "$OUT/$2.err"
    ncu -i "$1.ncu-rep" --page raw --csv > "$OUT/$2.raw.csv" 2>> "$OUT/$2.err"
    ncu -i "$1.ncu-rep" --page source --csv --print-source sass 2>> "$OUT/$2.err" | gzip > "$OUT/$2.source_sass.csv.gz"
    ls -la "$1.ncu-rep"
    if [ "$(du -sm "$OUT" | cut -f1)" -gt 55 ]; then rm -f "$1.ncu-rep"; echo "dropped $1.ncu-rep (size cap)"; fi
  fi
}
timeout 300 $B1 > "$OUT/plain1_$TAG.log" 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on \
    -k "regex:k_direct_chirp" -s 1 -c 1 -o "$OUT/prof_k3_cfg1_$TAG" $B1 > "$OUT/ncu_k3_1_$TAG.log" 2>&1; echo "ncu_k3_1=$?"
summarise "$OUT/prof_k3_cfg1_$TAG" "ncu_k3chirp_cfg1_$TAG"
timeout 900 $B4 > "$OUT/plain4b_$TAG.log" 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on \
    -k "regex:k_direct_chirp" -s 2 -c 1 -o "$OUT/prof_k3_cfg4_$TAG" $B4 > "$OUT/ncu_k3_$TAG.log" 2>&1; echo "ncu_k3_4=$?"
summarise "$OUT/prof_k3_cfg4_$TAG" "ncu_k3chirp_cfg4_$TAG"
du -sm "$OUT"
