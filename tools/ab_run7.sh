#!/bin/bash
# A/B: Adam streaming cache hints (default build) vs plain loads / stores, C2 step N=1
one() {
  env "$@" timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); print(round(d["value"]), round(d["ms_per_step"],4), d["hbm_kernels"]["adam"]["achieved_gbps"])' 2>&1 | tail -1)" >> gpurun_out/ab7.txt
}
for rep in 1 2 3; do
  one HP_X=stream
  one HP_LIB_VARIANT=plainadam
done
