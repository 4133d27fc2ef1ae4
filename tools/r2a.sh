set -u
mkdir -p gpurun_out
export WCGH_PARITY_LOG=gpurun_out/r2_parity.jsonl
rm -f $WCGH_PARITY_LOG
timeout 1500 python -m pytest tests -x -q -m gpu --durations=30 > gpurun_out/r2_gputests.log 2>&1; echo "pytest=$?"
tail -5 gpurun_out/r2_gputests.log
timeout 900 python bench.py --steps 3 --warmup 1 > gpurun_out/r2_bench_short.json 2> gpurun_out/r2_bench_short.err; echo "bench=$?"
WCGH_BENCH_SAME_DEVICE=1 WCGH_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --config 1 --steps 3 --warmup 1 --no-extra > gpurun_out/r2_bench_2rank.json 2> gpurun_out/r2_bench_2rank.err; echo "bench2=$?"
