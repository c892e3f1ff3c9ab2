#!/bin/bash
# A/B: Adam grid cap (CTAs per update launch) at N=1
one() {
  env "$@" timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); print(round(d["value"]), round(d["ms_per_step"],4), d["hbm_kernels"]["adam"])' 2>&1 | tail -1)" >> gpurun_out/ab5.txt
}
for rep in 1 2; do
  one HP_ADAM_GRID=0
  one HP_ADAM_GRID=148
  one HP_ADAM_GRID=296
  one HP_ADAM_GRID=74
done
