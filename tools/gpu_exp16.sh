# 16-view step timing per build variant (VARIANTS ';'-separated), 3 worker streams
set -x
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for F in "" "${VS[@]}"; do
  echo "=== variant: ${F:-baseline}"
  SS_NVCC_FLAGS="$F" python -c "from paper_2605_05876_b200 import build as b; b.build(force=True)" || exit 1
  NVIEWS=16 STREAMS=${STREAMS:-1,3} python tools/kernel_timing.py 2>&1 | grep -E "train_|chain|preprocess|bin_sort|sum|streams="
done
SS_NVCC_FLAGS="" python -c "from paper_2605_05876_b200 import build as b; b.build(force=True)"
