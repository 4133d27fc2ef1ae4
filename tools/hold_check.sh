python tools/hold_error.py > gpurun_out/s5_hold_error.jsonl 2> gpurun_out/s5_hold_error.err; echo hold_err=$?
timeout 600 python -m pytest tests/test_gpu_direct_forms.py -x -q -m gpu > gpurun_out/s5_tests_forms.log 2>&1; echo forms=$? $(tail -1 gpurun_out/s5_tests_forms.log)
WCGH_PARITY_LOG=gpurun_out/s5_parity.jsonl timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_fullplane.py -x -q -m gpu > gpurun_out/s5_tests_cfg.log 2>&1; echo cfg=$? $(tail -1 gpurun_out/s5_tests_cfg.log)
