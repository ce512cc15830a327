set -x
TAG=${TAG:-r1}
python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "ss_step/" \
    -k regex:"${FULLK:-raster}" -c ${FULLC:-2} -o gpurun_out/prof_$TAG python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
