# round refresh: bench (both arms), launch list with DRAM bytes, ncu --set full of the main kernels
set -x
TAG=${TAG:-r2f}
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -2 gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
TAG=$TAG bash tools/gpu_prof2.sh
