set -x
timeout 900 python -m pytest tests -q -m gpu -x -k "knn or refine or boundary" 2>&1 | tail -4
STEPS=4 timeout 600 python tools/knn_diag.py 2>&1 | tail -4
timeout 600 python tools/refine_timing.py 2>&1 | tail -8
