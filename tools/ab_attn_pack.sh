#!/bin/bash
# C3 attention packing (consecutive short pairs share a 128-row tile) vs one pair per CTA
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/abp_tests.log 2>&1; echo EXIT $? >> gpurun_out/abp_tests.log
one() {
  env "$@" timeout 600 python bench.py --workload c3 --steps 20 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); a=d["roofline"]["attention"]; print(round(d["value"]), round(d["ms_per_step"],4), "attn replay", round(a["replay_ms_per_step"],4), "in-step", round(a["ms_per_step"],4), "frac", round(a["frac"],4))' 2>&1 | tail -1)" >> gpurun_out/abp.txt
}
for rep in 1 2; do
  one HP_X=pack
  one HP_ATTN_PACK=0
done
