# build variants (SS_NVCC_FLAGS) and time the per-stage kernels: VARIANTS="a;b"
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for F in "${VS[@]}"; do
  echo "=== variant: ${F:-baseline}"
  SS_NVCC_FLAGS="$F" python -c "from paper_2605_05876_b200 import build as b; b.build(force=True)" || exit 1
  STREAMS=${STREAMS:-1,3} python tools/kernel_timing.py 2>&1 | grep -v Warn
done
SS_NVCC_FLAGS="" python -c "from paper_2605_05876_b200 import build as b; b.build(force=True)"
