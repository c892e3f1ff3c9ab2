#!/bin/bash
# 4-GPU step time under NCCL algorithm / CTA-count settings (bench value pass only)
for cfg in ${CFGS:-"" "NCCL_ALGO=allreduce:nvls" "NCCL_ALGO=allreduce:nvlstree" "NCCL_ALGO=allreduce:nvls NCCL_NVLS_NCHANNELS=16"}; do
  env $cfg timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NG:-4} --master-addr 127.0.0.1 \
    --master-port 29520 bench.py --gpus ${NG:-4} --steps 20 --no-cpu-baseline --no-e2e > /tmp/b.json 2>/tmp/b.err
  echo "[$cfg] $(tail -1 /tmp/b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],3))' 2>&1 | tail -1)"
done
