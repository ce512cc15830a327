set -x
TAG=${TAG:-r1}
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -2 gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "ss_step/" -c 2000 --csv \
    --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
NVIEWS=2 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "ss_step/" \
    -k regex:"splat_bwd|raster_fwd|chain|scatter|tile_sort|preprocess" -c 8 -o gpurun_out/prof_$TAG python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
