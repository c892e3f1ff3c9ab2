#!/bin/bash
# N = 1 bucket size (update granularity only): 150 / 200 / 300 / 500 MB
one() {
  timeout 300 python bench.py --steps 40 --bucket-mb $1 --no-cpu-baseline --no-e2e --no-same-config > /tmp/o.json 2>/tmp/o.err
  echo "[bucket $1] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); print(round(d["value"]), round(d["ms_per_step"],4))' 2>&1 | tail -1)" >> gpurun_out/abb.txt
}
for rep in 1 2; do for b in 150 200 300 500; do one $b; done; done
