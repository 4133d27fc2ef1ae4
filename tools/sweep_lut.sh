mkdir -p gpurun_out
for v in "8,4,2" "16,2,2" "16,2,4" "8,2,4" "12,2,4"; do
  for ch in 48 24; do
    r=$(WCGH_LUT_VARIANT=$v WCGH_LUT_CHUNKS=$ch timeout 300 python bench.py --config 2 --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.2f ms  frac %.3f' % (d['ms_per_step'], d['roofline']['frac']))" 2>&1)
    echo "variant=$v chunks=$ch cfg2: $r"
  done
done
