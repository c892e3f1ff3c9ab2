#!/bin/bash
# A/B: split-K cap of the weight-gradient GEMMs (wgrad stream) at N=1
one() {
  env "$@" timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); print(round(d["value"]), round(d["ms_per_step"],4))' 2>&1 | tail -1)" >> gpurun_out/ab3.txt
}
for rep in 1 2; do
  one HP_WGRAD_SPLIT_MAX=0
  one HP_WGRAD_SPLIT_MAX=1
  one HP_WGRAD_SPLIT_MAX=2
  one HP_WGRAD_STREAM=0
done
