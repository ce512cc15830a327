# smoke() on the GPU, then bench.py under torchrun (1 rank, NCCL forced): stdout must be the JSON line only
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')"
SS_COLLECTIVES=force timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29555 bench.py --gpus 1 --steps 3 --warmup 3 --no-configs --no-cpu > gpurun_out/bench_nccl2.json 2> gpurun_out/bench_nccl2.err
echo "bench rc=$?"; wc -l gpurun_out/bench_nccl2.json
python -c "import json; d=json.loads(open('gpurun_out/bench_nccl2.json').read()); print(d['value'], d['e2e']['value'], d['config']['collective'], d['per_step_fixed_ms']['allreduce'])"
