#!/bin/bash
# N = 2 / 4 A/B: forward GEMMs on every SM (default) vs the 140-SM cap in forward too (HP_GEMM_SMS_FWD=140)
run() {
  env $2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) bench.py --gpus $1 --no-e2e --no-cpu-baseline \
    --no-same-config --no-loss-check 2>/dev/null | python -c "import json,sys;j=json.loads(sys.stdin.read());a=j['allreduce'];print('N $1 $2', round(j['value'],1), round(j['ms_per_step'],3), 'exposed', round(a['exposed_ms'],3), 'nocomm', round(a['ms_per_step_without_grad_allreduce'],3))"
}
for rep in 1 2; do
  run 2 HP_X=fwdall
  run 2 HP_GEMM_SMS_FWD=140
done
for rep in 1 2; do
  run 4 HP_X=fwdall
  run 4 HP_GEMM_SMS_FWD=140
done
