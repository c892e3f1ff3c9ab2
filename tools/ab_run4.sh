#!/bin/bash
# A/B: row-sparse word-embedding exchange at N=2 and N=4
for NG in 4 2; do
for sp in 1 0 1 0; do
  HP_SPARSE_EMB=$sp timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus $NG --steps 30 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
  echo "[sparse=$sp] N=$NG $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); a=d["allreduce"]; print(round(d["value"]), round(d["ms_per_step"],4), "bus", round(a["bus_gbps"]), "alone", round(a["ms_alone"],3), "exposed", round(a["exposed_ms"],3), "nocomm", round(a["ms_per_step_without_grad_allreduce"],3))' 2>&1 | tail -1)" >> gpurun_out/ab4.txt
done
done
