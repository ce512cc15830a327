# variant timings (gpu_exp.sh) then a parity subset on the default build
set -x
VARIANTS="${VARIANTS}" bash tools/gpu_exp.sh > gpurun_out/exp_${TAG:-r2g}.log 2>&1
cat gpurun_out/exp_${TAG:-r2g}.log | grep -v "^+"
timeout 900 python -m pytest tests -q -m gpu -x ${QK:+-k "$QK"} 2>&1 | tail -5
