# end-of-session refresh: GPU tests, bench (both arms), launch list + DRAM bytes, ncu --set full of the main kernels
set -x
TAG=${TAG:-r2i}
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/gputest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_$TAG.log
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
TAG=$TAG bash tools/gpu_prof2.sh
ls -la gpurun_out | tail -12
