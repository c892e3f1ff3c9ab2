#!/bin/bash
# C4 long-attention forward with 8 softmax warps (two per lane quarter, key blocks split by parity) vs 4 (prefl = previous HEAD)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/abl_tests.log 2>&1; echo EXIT $? >> gpurun_out/abl_tests.log
one() {
  env "$@" timeout 600 python bench.py --workload c4 --steps 10 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); a=d["roofline"]["attention"]; print(round(d["value"],1), round(d["ms_per_step"],3), "attn replay", round(a["replay_ms_per_step"],3), "in-step", round(a["ms_per_step"],3))' 2>&1 | tail -1)" >> gpurun_out/abl.txt
}
for rep in 1 2; do
  one HP_X=new
  one HP_LIB_VARIANT=prefl
done
