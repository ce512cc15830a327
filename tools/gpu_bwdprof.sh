# launch list of one profiled step + ncu --set full of the record backward
set -x
export NVIEWS=${NVIEWS:-2}
python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "ss_step/" --csv \
    --log-file gpurun_out/bwd_launches.csv python tools/profile_step.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "ss_step/" \
    -k regex:"${FULLK:-splat_bwd}" -c ${FULLC:-1} -o gpurun_out/prof_${TAG:-bwd} -f python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
