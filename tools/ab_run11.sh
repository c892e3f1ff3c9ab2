#!/bin/bash
# A/B: LayerNorm rows per CTA (backward 32 vs 16; forward 2 vs 1 rows per warp), C2 N=1
timeout 600 env HP_LIB_VARIANT=ln16f1 python -m pytest tests/test_gpu_engine.py -x -q -k "bert or graph" > gpurun_out/ab11_tests.log 2>&1; echo EXIT $? >> gpurun_out/ab11_tests.log
one() {
  env "$@" timeout 300 python bench.py --steps 40 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); print(round(d["value"]), round(d["ms_per_step"],4), d["breakdown_ms_per_step"]["layernorm"])' 2>&1 | tail -1)" >> gpurun_out/ab11.txt
}
for rep in 1 2 3; do
  one HP_X=base
  one HP_LIB_VARIANT=lnb16
  one HP_LIB_VARIANT=ln16f1
done
