#!/usr/bin/env bash
# K4 chunk-kernel window shapes (needs a build with WCGH_NVCC_EXTRA=-DWCGH_LUT_SWEEP):
# config 2 LUT kernel time and FP32 fraction per shape R,PX,D,W and gap threshold.
set -u
OUT=${OUT:-gpurun_out}; TAG=${TAG:-s5b}
mkdir -p "$OUT"
for v in ${VARIANTS:-"16,2,2,4" "16,2,1,4" "16,2,3,4" "12,2,2,4" "16,1,2,4" "16,2,2,2" "24,1,2,2" "32,1,2,2" "24,2,2,2" "20,2,2,2"}; do
  for g in ${GAPS:-4 16}; do
    for cfg in ${CFGS:-2}; do
    r=$(WCGH_LUT_VARIANT=$v WCGH_LUT_GAP=$g timeout 300 python bench.py --config $cfg --method lut --steps 5 --warmup 3 --no-cpu-baseline --no-extra 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('%.3f ms  kernel %.3f ms  frac %.4f' % (d['ms_per_step'], r['kernel_ms'], r['frac']))" 2>&1)
    echo "variant=$v gap=$g cfg$cfg lut: $r"
    done
  done
done | tee "$OUT/k4chunk_sweep_$TAG.txt"
