# A/B of the current tree against _old (a worktree of an earlier commit): stage timings, configs 3 and 1, photometric step; parity subset
set -x
NVIEWS=16 timeout 600 python tools/kernel_timing.py 2>&1 | head -9
(cd _old && NVIEWS=16 timeout 600 python tools/kernel_timing.py 2>&1 | head -9)
NVIEWS=16 STREAMS=3 LOSS=photometric timeout 600 python tools/kernel_timing.py 2>&1 | tail -1
(cd _old && NVIEWS=16 STREAMS=3 LOSS=photometric timeout 600 python tools/kernel_timing.py 2>&1 | tail -1)
timeout 600 python tools/config_timing.py 3 1
(cd _old && timeout 600 python tools/config_timing.py 3 1)
timeout 1500 python -m pytest tests -q -m gpu -x -k "${QK:-parity or fullsize or properties or train_step or boundary}" 2>&1 | tail -4
