# round-2 session-2 check: GPU tests, stage timing, KNN/refine timing, band-order variants
set -x
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -6
timeout 600 python tools/refine_timing.py 2>&1 | tail -12
VARIANTS="${VARIANTS:--DSS_BAND_H=4096;-DSS_TICKET_ROUNDS=8;-DSS_BAND_H=128}" timeout 1500 bash tools/gpu_exp.sh 2>&1 | grep -v "^+"
