#!/bin/bash
# Precision variants of the record backward on the photometric step:
# VARIANTS="flags1;flags2;..." (empty entry = baseline)
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for F in "${VS[@]}"; do
  echo "=== variant: ${F:-baseline}"
  SS_NVCC_FLAGS="$F" python -c "from paper_2605_05876_b200 import build as b; b.build(force=True)" || exit 1
  python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "photometric_step_full_size or training_gradients_full_size" 2>&1 | grep -E "passed|failed|AssertionError: config" | cut -c1-400
  python tools/grad_outliers.py 2 --records --photometric 793178 2>&1 | grep -A4 "^793178" | tail -2
  NVIEWS=16 STREAMS=1 python tools/kernel_timing.py 2>&1 | grep -E "train_backward|sum"
done
SS_NVCC_FLAGS="" python -c "from paper_2605_05876_b200 import build as b; b.build(force=True)"
