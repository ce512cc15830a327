set -x
python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "ss_step/" -c 2000 --csv \
    --log-file gpurun_out/launches_r1a.csv python tools/profile_step.py > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "ss_step/" \
    -k regex:raster -c 2 -o gpurun_out/prof_raster_r1a python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "ss_step/" \
    -k regex:"chain|preprocess|tile_sort" -c 3 -o gpurun_out/prof_other_r1a python tools/profile_step.py > gpurun_out/ncu_full2.log 2>&1
echo "full2 rc=$?"
tail -3 gpurun_out/ncu_full.log
