B="python bench.py --config 4 --method fft --steps 1 --warmup 1 --no-cpu-baseline --no-extra"
$B > gpurun_out/plain_fft.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fft_cfg4.csv $B > /dev/null 2>&1; echo l=$?
$B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:k_fft_rows|k_transpose" -s 6 -c 6 -o gpurun_out/prof_fft_cfg4 $B > gpurun_out/ncu_fft.log 2>&1; echo f=$?
