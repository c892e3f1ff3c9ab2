#!/bin/bash
# N = 4 A/B: GEMM SM budget x bucket size (C2, value pass + allreduce figures)
run() {
  env HP_GEMM_SMS=$1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 --bucket-mb $2 --no-e2e --no-cpu-baseline \
    --no-same-config --no-loss-check 2>/dev/null | python -c "import json,sys;j=json.loads(sys.stdin.read());a=j['allreduce'];print('sms $1 bucket $2', round(j['value'],1), round(j['ms_per_step'],3), 'exposed', round(a['exposed_ms'],3), 'nocomm', round(a['ms_per_step_without_grad_allreduce'],3))"
}
for rep in 1 2; do
  for cfg in "140 50" "132 50" "124 50" "140 100" "132 100" "140 25"; do run $cfg; done
done
