#!/bin/bash
# A/B matrix: PDL on/off at N=1, bucket size and NCCL settings at N=NG (4)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo EXIT $? >> gpurun_out/ab_tests.log
for pdl in 1 0 1 0; do
  HP_PDL=$pdl timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/dev/null
  echo "pdl=$pdl $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); print(round(d["value"]), round(d["ms_per_step"],4), d["roofline"]["frac"])')" >> gpurun_out/ab.txt
done
NG=${NG:-4}
for cfg in "B=25" "B=50" "B=100" "B=25 NCCL_MIN_NCHANNELS=32" "B=50 NCCL_MIN_NCHANNELS=32" "B=25 NCCL_ALGO=allreduce:nvls" "B=100 NCCL_ALGO=allreduce:nvls"; do
  B=$(echo $cfg | sed 's/.*B=\([0-9]*\).*/\1/'); envs=$(echo $cfg | sed 's/B=[0-9]*//')
  env $envs timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $NG --steps 30 --bucket-mb $B --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
  echo "[$cfg] N=$NG $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); a=d["allreduce"]; print(round(d["value"]), round(d["ms_per_step"],4), "bus", round(a["bus_gbps"]), "alone", round(a["ms_alone"],3), "exposed", round(a["exposed_ms"],3))' 2>&1 | tail -1)" >> gpurun_out/ab.txt
done
