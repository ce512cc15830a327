# standalone per-kernel durations (serialised, ncu launch list) of one profiled step
set -x
TAG=${TAG:-q}
python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "ss_step/" -c 2000 --csv \
    --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
