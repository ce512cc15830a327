# timing experiments: rebuild with each switch set (VARIANTS, ';'-separated) and time the stages
set -x
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for F in "" "${VS[@]}"; do
  echo "=== variant: ${F:-baseline}"
  SS_NVCC_FLAGS="$F" python -c "from paper_2605_05876_b200 import build as b; b.build(force=True)" || exit 1
  NVIEWS=${NVIEWS:-8} python tools/kernel_timing.py 2>&1 | sed -n 1,9p
done
# restore the default build on exit (the stamp would force it anyway)
SS_NVCC_FLAGS="" python -c "from paper_2605_05876_b200 import build as b; b.build(force=True)"
