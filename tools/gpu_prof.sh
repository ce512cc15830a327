# ncu --set full (with source) of the main kernels of one profiled step (NVIEWS views)
set -x
TAG=${TAG:-p}
export NVIEWS=${NVIEWS:-2}
python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "ss_step/" \
    -k regex:"${FULLK:-splat_bwd|raster_fwd|chain|scatter|tile_sort|preprocess}" -c ${FULLC:-6} -o gpurun_out/prof_$TAG python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
