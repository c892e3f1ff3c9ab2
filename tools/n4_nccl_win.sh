#!/bin/bash
# N = 2 / 4 A/B: gradient buffer as a symmetric NCCL window (HP_NCCL_WIN=1) vs plain cudaMalloc
run() {
  env $2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) bench.py --gpus $1 --no-e2e --no-cpu-baseline \
    --no-same-config --no-loss-check 2>gpurun_out/nw_err_$1.log | python -c "import json,sys;j=json.loads(sys.stdin.read());a=j['allreduce'];print('N $1 $2', round(j['value'],1), round(j['ms_per_step'],3), 'exposed', round(a['exposed_ms'],3), 'alone', round(a['ms_alone'],3), 'busbw', round(a['bus_gbps'],1))"
}
for rep in 1 2; do
  run 2 HP_X=plain
  run 2 HP_NCCL_WIN=1
  run 4 HP_X=plain
  run 4 HP_NCCL_WIN=1
done
