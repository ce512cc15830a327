# timing experiments: rebuild with each switch set and time the stages
for F in "" "-DSS_EXP_NO_SHADE" "-DSS_EXP_NO_MARGIN" "-DSS_EXP_NO_REDUCE" "-DSS_EXP_NO_PHASE2"; do
  echo "=== variant: ${F:-baseline}"
  SS_NVCC_FLAGS="$F" python -c "from paper_2605_05876_b200 import build as b; b.build(force=True)" || exit 1
  NVIEWS=8 python tools/kernel_timing.py 2>&1 | sed -n 1,6p
done
