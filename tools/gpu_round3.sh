# session-3 refresh: GPU tests, then the bench (both arms)
set -x
TAG=${TAG:-r2h}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/gputest_$TAG.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/gputest_$TAG.log
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
