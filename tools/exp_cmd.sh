set -x
STREAMS=1,3 python tools/kernel_timing.py 2>&1 | grep -v Warn
MORTON=1 STREAMS=1,3 python tools/kernel_timing.py 2>&1 | grep -v Warn
SS_NVCC_FLAGS="-DSS_GW_F32" python -c "from paper_2605_05876_b200 import build as b; b.build(force=True)"
STREAMS=1,3 python tools/kernel_timing.py 2>&1 | grep -v Warn
python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -x 2>&1 | tail -3
python -c "from paper_2605_05876_b200 import build as b; b.build(force=True)"
