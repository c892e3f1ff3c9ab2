#!/bin/bash
# N = 4 (and 2) A/B: split word-embedding update (HP_EMB_SPLIT=1: rows outside the
# batch's ids updated during backward) vs default
run() {
  env $2 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) bench.py --gpus $1 --no-e2e --no-cpu-baseline \
    --no-same-config --no-loss-check 2>/dev/null | python -c "import json,sys;j=json.loads(sys.stdin.read());a=j['allreduce'];print('N $1 $2', round(j['value'],1), round(j['ms_per_step'],3), 'exposed', round(a['exposed_ms'],3), 'alone', round(a['allreduce_alone_ms'] if 'allreduce_alone_ms' in a else -1,3), 'nocomm', round(a['ms_per_step_without_grad_allreduce'],3))"
}
for rep in 1 2; do
  for cfg in "HP_X=0" "HP_EMB_SPLIT=1"; do run 4 $cfg; done
done
for cfg in "HP_X=0" "HP_EMB_SPLIT=1"; do run 2 $cfg; done
