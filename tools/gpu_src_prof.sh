# source-level ncu capture (one launch each) of the main kernels of one step
set -x
TAG=${TAG:-r2e}
NVIEWS=1 python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 || exit 1
NVIEWS=1 timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "ss_step/" \
    -k regex:"${FULLK:-splat_bwd|raster_fwd|chain_kernel|preprocess_kernel}" -c ${FULLC:-4} \
    -o gpurun_out/src_$TAG -f python tools/profile_step.py > gpurun_out/ncu_src.log 2>&1
echo "src rc=$?"
