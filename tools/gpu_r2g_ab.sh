# NCCL self-test with full output; config-3 A/B (HEAD vs _old = 646e8cb)
set -x
env | grep -i nccl
SS_COLLECTIVES=force timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29544 tests/nccl_selftest.py > gpurun_out/nccl_selftest.out 2> gpurun_out/nccl_selftest.err
echo "selftest rc=$?"; cat gpurun_out/nccl_selftest.out; tail -30 gpurun_out/nccl_selftest.err
timeout 600 python tools/config_timing.py 3
(cd _old && timeout 600 python tools/config_timing.py 3)
timeout 600 python tools/config_timing.py 3
