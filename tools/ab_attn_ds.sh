#!/bin/bash
# A/B: attention backward computes dS before dV's MMA completes (held packed in registers) vs after (base)
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention or attn" > gpurun_out/abd_tests.log 2>&1; echo EXIT $? >> gpurun_out/abd_tests.log
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q -k "bert and (bf16 or graph)" >> gpurun_out/abd_tests.log 2>&1; echo EXIT $? >> gpurun_out/abd_tests.log
one() {
  env "$@" timeout 300 python bench.py --steps 40 --no-cpu-baseline --no-e2e --no-same-config > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); r=d["roofline"]; a=r["attention"]; print(round(d["value"]), round(d["ms_per_step"],4), "attn replay", round(a["replay_ms_per_step"],4), "in-step", round(a["ms_per_step"],4))' 2>&1 | tail -1)" >> gpurun_out/abd.txt
}
for rep in 1 2 3; do
  one HP_X=new
  one HP_LIB_VARIANT=base
done
