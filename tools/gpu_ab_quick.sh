# A/B stage timing against _old, then a parity subset
set -x
NVIEWS=16 timeout 600 python tools/kernel_timing.py 2>&1 | head -9
(cd _old && NVIEWS=16 timeout 600 python tools/kernel_timing.py 2>&1 | head -9)
timeout 1500 python -m pytest tests -q -m gpu -x -k "${QK:-parity or fullsize or train_step or boundary}" 2>&1 | tail -3
