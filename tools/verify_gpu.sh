#!/usr/bin/env bash
# One GPU pass: smoke, the whole -m gpu suite (parity log), a short default bench.
set -u
OUT=${OUT:-gpurun_out}
TAG=${TAG:-v}
mkdir -p "$OUT"
export WCGH_PARITY_LOG=$OUT/parity_$TAG.jsonl
rm -f $WCGH_PARITY_LOG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > "$OUT/gpu_$TAG.txt" 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke_$TAG.log" 2>&1; echo "smoke=$?"
timeout ${PYT_TIMEOUT:-1800} python -m pytest tests -x -q -m gpu --durations=25 ${PYT_ARGS:-} > "$OUT/gputests_$TAG.log" 2>&1; echo "pytest=$?"
tail -3 "$OUT/gputests_$TAG.log"
if [ -z "${SKIP_BENCH:-}" ]; then
timeout 900 python bench.py --steps 3 --warmup 3 > "$OUT/bench_$TAG.json" 2> "$OUT/bench_$TAG.err"; echo "bench=$?"
fi
