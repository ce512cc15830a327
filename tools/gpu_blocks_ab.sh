# block lists on/off (SS_BLOCK_LISTS), stage timings and 3-stream step; then parity of the default (on)
set -x
for B in 1 0 1; do echo "=== SS_BLOCK_LISTS=$B"; SS_BLOCK_LISTS=$B NVIEWS=16 timeout 600 python tools/kernel_timing.py 2>&1 | head -9; done
timeout 1500 python -m pytest tests -q -m gpu -x -k "${QK:-fullsize or train_step or parity or nccl}" 2>&1 | tail -3
