IFS=';' read -ra VS <<< "${VARIANTS:-}"
for F in "${VS[@]}"; do
  echo "=== variant: ${F:-baseline}"
  SS_NVCC_FLAGS="$F" python -c "from paper_2605_05876_b200 import build as b; b.build(force=True)" || exit 1
  python tools/grad_outliers.py 2 > gpurun_out/go2v.log 2>&1; grep "step outliers" gpurun_out/go2v.log | head -8
  python tools/grad_outliers.py 3 > gpurun_out/go3v.log 2>&1; grep "step outliers" gpurun_out/go3v.log | head -8
  NVIEWS=16 STREAMS=1 python tools/kernel_timing.py 2>&1 | grep -E "train_backward|chain|sum"
done
SS_NVCC_FLAGS="" python -c "from paper_2605_05876_b200 import build as b; b.build(force=True)"
