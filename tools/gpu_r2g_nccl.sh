# NCCL self-test on one GPU: the pytest, then bench.py through torchrun (1 rank, SS_COLLECTIVES=force)
set -x
timeout 900 python -m pytest tests/test_gpu_nccl.py -q -x 2>&1 | tail -5
SS_COLLECTIVES=force timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/bench_nccl1.json 2> gpurun_out/bench_nccl1.err
echo "bench rc=$?"; tail -3 gpurun_out/bench_nccl1.err
python -c "import json; d=json.load(open('gpurun_out/bench_nccl1.json')); print(d['value'], d['e2e']['value'], d['config']['collective'])"
