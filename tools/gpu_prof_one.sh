# ncu --set full of kernels matching $K (one launch each, $C launches) in a 2-view profiled step
TAG=${TAG:-one}
NVIEWS=2 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "ss_step/" \
    -k regex:"$K" -c ${C:-2} -o gpurun_out/prof_$TAG -f python tools/profile_step.py > gpurun_out/ncu_$TAG.log 2>&1
echo "rc=$?"
