#!/bin/bash
# GPU suite, then A/B: layer-parity gradient slots (default) vs one slot, C2 step N=1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/ab8_tests.log 2>&1; echo EXIT $? >> gpurun_out/ab8_tests.log
one() {
  env "$@" timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); print(round(d["value"]), round(d["ms_per_step"],4))' 2>&1 | tail -1)" >> gpurun_out/ab8.txt
}
for rep in 1 2 3; do
  one HP_LAYER_SLOTS=2
  one HP_LAYER_SLOTS=1
done
