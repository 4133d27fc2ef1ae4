for v in 8,2,4,4 8,2,2,4 8,2,4,8 8,4,2,4; do
  WCGH_LUT_VARIANT=$v timeout 120 python bench.py --config 2 --method lut --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1 && \
  WCGH_LUT_VARIANT=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_lut_stage --log-file gpurun_out/stage_$v.csv python bench.py --config 2 --method lut --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  echo "done $v"
done
