#!/bin/bash
# embedding gradient: hot and small ids in one launch (new) vs two launches (prefin = 405bd79)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/abe2_tests.log 2>&1; echo EXIT $? >> gpurun_out/abe2_tests.log
one() {
  env "$@" timeout 300 python bench.py --steps 40 --no-cpu-baseline --no-e2e --no-same-config > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); print(round(d["value"]), round(d["ms_per_step"],4), "emb", d["breakdown_ms_per_step"]["embedding"], "launches/step", d["gpu_launches"]/d["steps"])' 2>&1 | tail -1)" >> gpurun_out/abe2.txt
}
for rep in 1 2 3; do
  one HP_X=new
  one HP_LIB_VARIANT=prefin
done
