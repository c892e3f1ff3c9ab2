#!/bin/bash
# A/B at N=4: NCCL channel caps / protocol for the gradient buckets
NG=${NG:-4}
for cfg in "X=1" "NCCL_MAX_NCHANNELS=16" "NCCL_MAX_NCHANNELS=8" "NCCL_PROTO=Simple" "X=1" "NCCL_MAX_NCHANNELS=16"; do
  env $cfg timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $NG --steps 30 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
  echo "[$cfg] N=$NG $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); a=d["allreduce"]; print(round(d["value"]), round(d["ms_per_step"],4), "bus", round(a["bus_gbps"]), "alone", round(a["ms_alone"],3), "exposed", round(a["exposed_ms"],3))' 2>&1 | tail -1)" >> gpurun_out/ab9.txt
done
