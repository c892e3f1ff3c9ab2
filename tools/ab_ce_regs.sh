#!/bin/bash
# label-smoothed CE: the row kept in registers between the two passes (new) vs re-read (prece = previous HEAD)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/abc_tests.log 2>&1; echo EXIT $? >> gpurun_out/abc_tests.log
one() {
  env "${@:2}" timeout 600 python bench.py --workload $1 --steps 20 --no-cpu-baseline --no-e2e --no-same-config > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); print(round(d["value"]), round(d["ms_per_step"],4), "heads", d["breakdown_ms_per_step"]["heads"])' 2>&1 | tail -1)" >> gpurun_out/abc.txt
}
for rep in 1 2; do
  one c3 HP_X=new
  one c3 HP_LIB_VARIANT=prece
  one c2 HP_X=new
  one c2 HP_LIB_VARIANT=prece
done
