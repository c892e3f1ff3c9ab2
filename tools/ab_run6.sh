#!/bin/bash
# A/B: cluster split-K (deterministic weight gradients) vs fp32-atomics split-K, C2 step N=1
one() {
  env "$@" timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); print(round(d["value"]), round(d["ms_per_step"],4))' 2>&1 | tail -1)" >> gpurun_out/ab6.txt
}
for rep in 1 2 3; do
  one HP_GEMM_CSPLIT=1
  one HP_GEMM_CSPLIT=0
done
