# round-2 profile: launch list of one 8-view step + ncu --set full of the
# main kernels (one launch each), reports -> gpurun_out/prof_$TAG.ncu-rep
set -x
TAG=${TAG:-r2a}
export NVIEWS=${NVIEWS:-8}
python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx \
    --nvtx-include "ss_step/" --csv --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > /dev/null 2>&1
echo "launch rc=$?"
NVIEWS=2 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "ss_step/" \
    -k regex:"splat_bwd|raster_fwd|chain_kernel|preprocess_kernel|tile_sort|^scatter_kernel|big_bwd" -c 8 \
    -o gpurun_out/prof_$TAG -f python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
