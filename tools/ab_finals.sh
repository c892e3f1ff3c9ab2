#!/bin/bash
# A/B: column-reduction finals batched into one launch per gradient bucket (new) vs one launch each (base)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/abf_tests.log 2>&1; echo EXIT $? >> gpurun_out/abf_tests.log
one() {
  env "$@" timeout 300 python bench.py --steps 40 --no-cpu-baseline --no-e2e --no-same-config > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); h=d["hbm_kernels"]["layernorm"]; print(round(d["value"]), round(d["ms_per_step"],4), "launches", d["gpu_launches"], "ln", h["launches_per_step"], d["breakdown_ms_per_step"]["layernorm"])' 2>&1 | tail -1)" >> gpurun_out/abf.txt
}
for rep in 1 2 3; do
  one HP_X=new
  one HP_LIB_VARIANT=base
done
