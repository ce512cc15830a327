set -x
SS_NVCC_FLAGS=-DSS_CTA_TIMING python -c "from paper_2605_05876_b200 import build as b; b.build()" || exit 1
python tools/tail_stats.py
SS_NVCC_FLAGS="" python -c "from paper_2605_05876_b200 import build as b; b.build()"
