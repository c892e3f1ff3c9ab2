#!/bin/bash
# A/B: PDL variants at N=1, separate update stream at N=4 (bucket sizes)
one() {  # env... -> value ms frac
  env "$@" timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); print(round(d["value"]), round(d["ms_per_step"],4))' 2>&1 | tail -1)" >> gpurun_out/ab2.txt
}
for rep in 1 2; do
  one HP_PDL=0
  one HP_PDL=1
  one HP_PDL=1 HP_LIB_VARIANT=notrig
  one HP_PDL=gemm
  one HP_PDL=ln,attn
  one HP_PDL=gemm HP_LIB_VARIANT=notrig
done
NG=${NG:-4}
for B in 25 50 100; do
  HP_PDL=0 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $NG --steps 30 --bucket-mb $B --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
  echo "[B=$B upd-stream] N=$NG $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); a=d["allreduce"]; print(round(d["value"]), round(d["ms_per_step"],4), "bus", round(a["bus_gbps"]), "alone", round(a["ms_alone"],3), "exposed", round(a["exposed_ms"],3))' 2>&1 | tail -1)" >> gpurun_out/ab2.txt
done
