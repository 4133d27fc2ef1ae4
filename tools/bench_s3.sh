#!/usr/bin/env bash
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-s3}
mkdir -p "$OUT"
SECONDS=0; timeout 1500 python bench.py > "$OUT/bench_default_$TAG.json" 2> "$OUT/bench_default_$TAG.err"; echo "bench=$? wall=$SECONDS"
SECONDS=0; timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/bench_ref_$TAG.json" 2> "$OUT/bench_ref_$TAG.err"; echo "ref=$? wall=$SECONDS"
