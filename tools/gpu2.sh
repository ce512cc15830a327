set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -25
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_r1a.json 2> gpurun_out/bench_r1a.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_r1a.err; cat gpurun_out/bench_r1a.json
