# quick iteration: gpu tests (or a -k subset), then per-stage kernel timing
set -x
timeout 900 python -m pytest tests -q -m gpu -x ${QK:+-k "$QK"} 2>&1 | tail -4
timeout 600 python tools/kernel_timing.py 2>&1 | tail -9
