# quick iteration: a -k subset of the GPU tests (QK), then the 16-view stage timing
set -x
timeout 1500 python -m pytest tests -q -m gpu -x ${QK:+-k "$QK"} 2>&1 | tail -4
NVIEWS=16 STREAMS=1,3 timeout 600 python tools/kernel_timing.py 2>&1 | grep -E "train_|chain|preprocess|bin_sort|sum|streams="
