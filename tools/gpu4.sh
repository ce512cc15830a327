# round-trip: smoke, GPU tests, bench, launch list (same workload as bench via tools/profile_step.py)
set -x
TAG=${TAG:-r1}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
if [ "${PROFILE:-1}" = "1" ]; then
python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "ss_step/" -c 2000 --csv \
    --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
fi
if [ "${FULL:-0}" = "1" ]; then
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "ss_step/" \
    -k regex:"${FULLK:-raster}" -c ${FULLC:-2} -o gpurun_out/prof_$TAG python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
fi
