# full gpu test suite + one bench line (no cpu baseline)
set -x
TAG=${TAG:-c}
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -6
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
