# K4 shape sweep (WCGH_LUT_VARIANT="R,PX,D,W"), configs 2 and 1: ms and FP32 fraction
mkdir -p gpurun_out
for v in ${VARIANTS:-"8,2,2,4" "8,2,1,4" "8,2,3,4" "8,2,4,4" "8,2,2,8" "8,4,2,4"}; do
  for cfg in ${CFGS:-2 1}; do
    r=$(WCGH_LUT_VARIANT=$v timeout 300 python bench.py --config $cfg --method lut --steps 5 --warmup 2 --no-cpu-baseline --no-extra 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('%.2f ms  kernel %.3f ms  frac %.4f' % (d['ms_per_step'], r['kernel_ms'], r['frac']))" 2>&1)
    echo "variant=$v kernel=${WCGH_LUT_KERNEL:-stream} cfg$cfg lut: $r"
  done
done
