#!/bin/bash
# LayerNorm backward: 28 rows per CTA (147 CTAs at C2, default) vs 32 (128 CTAs, ln32)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/abln_tests.log 2>&1; echo EXIT $? >> gpurun_out/abln_tests.log
one() {
  env "$@" timeout 300 python bench.py --steps 40 --no-cpu-baseline --no-e2e --no-same-config > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); print(round(d["value"]), round(d["ms_per_step"],4), "ln", d["breakdown_ms_per_step"]["layernorm"])' 2>&1 | tail -1)" >> gpurun_out/abln.txt
}
for rep in 1 2 3; do
  one HP_X=rows28
  one HP_LIB_VARIANT=ln32
done
