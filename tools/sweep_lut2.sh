mkdir -p gpurun_out
for rep in 1 2; do
for v in "8,4,2,4" "8,4,3,4"; do
  for cfg in 2; do
    r=$(WCGH_LUT_VARIANT=$v timeout 300 python bench.py --config $cfg --method lut --steps 5 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.2f ms  frac %.3f clk %s' % (d['ms_per_step'], d['roofline']['frac'], d['clocks']))" 2>&1)
    echo "rep=$rep variant=$v cfg$cfg lut: $r"
  done
done
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
