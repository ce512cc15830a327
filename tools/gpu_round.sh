set -x
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
timeout 1200 python bench.py > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_r2d.err
