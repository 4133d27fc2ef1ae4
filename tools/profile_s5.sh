#!/usr/bin/env bash
# Session-5 K4 pass (parameter-block form, k_lut_chunk) at config 2, LUT method:
#   1. launch list of the bench command (device time per launch);
#   2. ncu --set full (+source) of two B = 1 chunk launches;
#   3. LUT-method bench lines at configs 2, 1 and 4 (kernel ms, FP32 fraction).
# Every ncu command runs only after the identical plain command exited 0.
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-s5}
mkdir -p "$OUT"
B2="python bench.py --config 2 --method lut --steps 1 --warmup 1 --no-cpu-baseline --no-extra"
timeout 300 $B2 > "$OUT/plain2_$TAG.log" 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches_cfg2_$TAG.csv" $B2 > "$OUT/ncu_l2_$TAG.log" 2>&1; echo "ncu_launch=$?"
timeout 300 $B2 > "$OUT/plain2b_$TAG.log" 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on \
    --kernel-name-base demangled -k "regex:k_lut_chunk<\\(int\\)1," -s 6 -c 2 \
    -o "$OUT/prof_k4chunk_$TAG" $B2 > "$OUT/ncu_k4chunk_$TAG.log" 2>&1; echo "ncu_k4=$?"
for cfg in 2 1 4; do
  timeout 600 python bench.py --config $cfg --method lut --steps 5 --warmup 3 --no-cpu-baseline --no-extra > "$OUT/b${cfg}_lut_$TAG.json" 2> "$OUT/b${cfg}_lut_$TAG.err"
  python -c "
import json
d=json.loads(open('$OUT/b${cfg}_lut_$TAG.json').read().strip().splitlines()[-1]); r=d['roofline']
print('cfg$cfg lut: %.3f ms/holo  kernel %.3f ms  frac %.4f' % (d['ms_per_step'], r['kernel_ms'], r['frac']))"
done | tee "$OUT/k4_lut_configs_$TAG.txt"
