#!/bin/bash
# A/B at N=4: gradient buffer registered with NCCL (ncclMemAlloc + ncclCommRegister)
NG=${NG:-4}
for cfg in "HP_NCCL_REG=1" "HP_NCCL_REG=0" "HP_NCCL_REG=1" "HP_NCCL_REG=0"; do
  env $cfg timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus $NG --steps 30 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
  echo "[$cfg] N=$NG $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); a=d["allreduce"]; print(round(d["value"]), round(d["ms_per_step"],4), "exposed", round(a["exposed_ms"],3), "nocomm", round(a["ms_per_step_without_grad_allreduce"],3))' 2>&1 | tail -1)" >> gpurun_out/ab10.txt
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29582 -m pytest tests/test_gpu_multi.py -x -q -k c1_w2 > gpurun_out/ab10_test.log 2>&1
