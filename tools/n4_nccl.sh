#!/bin/bash
# N = 4 A/B: NCCL channel caps with the GEMM SM budget (C2)
run() {
  env HP_GEMM_SMS=$1 $2 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 --no-e2e --no-cpu-baseline \
    --no-same-config --no-loss-check 2>/dev/null | python -c "import json,sys;j=json.loads(sys.stdin.read());a=j['allreduce'];print('sms $1 $2', round(j['value'],1), round(j['ms_per_step'],3), 'exposed', round(a['exposed_ms'],3), 'alone', round(a['ms_alone'],3), 'busbw', round(a['bus_gbps'],1))"
}
for rep in 1 2; do
  run 140 "HP_X=0"
  run 140 "NCCL_MAX_NCHANNELS=8"
  run 140 "NCCL_MAX_NCHANNELS=16"
  run 132 "NCCL_MAX_NCHANNELS=16"
  run 140 "NCCL_ALGO=Tree"
done
