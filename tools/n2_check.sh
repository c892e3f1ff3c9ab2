#!/bin/bash
# N = 2: HEAD vs prefin (405bd79), two rounds
run() {
  env $1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) bench.py --gpus 2 --no-e2e --no-cpu-baseline \
    --no-same-config --no-loss-check 2>/dev/null | python -c "import json,sys;j=json.loads(sys.stdin.read());a=j['allreduce'];print('$1', round(j['value'],1), round(j['ms_per_step'],3), 'exposed', round(a['exposed_ms'],3), 'nocomm', round(a['ms_per_step_without_grad_allreduce'],3))"
}
for rep in 1 2; do
  run HP_X=head
  run HP_LIB_VARIANT=prefin
done
