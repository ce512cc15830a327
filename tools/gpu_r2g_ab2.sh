# after the 64-B pixel header: NCCL self-test pytest, config-3 A/B vs _old, config-2 stage timing, parity subset
set -x
timeout 900 python -m pytest tests/test_gpu_nccl.py -q -x 2>&1 | tail -3
timeout 600 python tools/config_timing.py 3 1
(cd _old && timeout 600 python tools/config_timing.py 3 1)
NVIEWS=16 timeout 600 python tools/kernel_timing.py 2>&1 | head -9
timeout 1500 python -m pytest tests -q -m gpu -x -k "fullsize or train_step or record_backward or photometric or boundary or properties or parity" 2>&1 | tail -4
