# quick iteration: the training-path parity tests + one bench line
set -x
TAG=${TAG:-q}
timeout 600 python -m pytest tests -q -m gpu -x -k "${QK:-train or backward}" 2>&1 | tail -4
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
