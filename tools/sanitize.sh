# compute-sanitizer passes over tools/sanitize_step.py; summaries -> gpurun_out/sanitize_*.txt
CS=/usr/local/cuda/bin/compute-sanitizer
for T in memcheck racecheck synccheck initcheck; do
  timeout 1500 $CS --tool $T --print-limit 20 --error-exitcode 9 python tools/sanitize_step.py > gpurun_out/sanitize_$T.txt 2>&1
  echo "$T rc=$?" >> gpurun_out/sanitize_rc.txt
done
tail -3 gpurun_out/sanitize_*.txt; cat gpurun_out/sanitize_rc.txt
