#!/bin/bash
# GPU suite and N = 1 A/B vs prefin (405bd79): C2 step + attention replay; C3 line
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/rv_tests.log 2>&1; echo EXIT $? >> gpurun_out/rv_tests.log
one() {
  env "$@" timeout 300 python bench.py --steps 40 --no-cpu-baseline --no-e2e --no-same-config > /tmp/o.json 2>/tmp/o.err
  echo "N1 [$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); a=d["roofline"]["attention"]; print(round(d["value"]), round(d["ms_per_step"],4), "attn replay", round(a["replay_ms_per_step"],4), "ln kernels", d["hbm_kernels"]["layernorm"]["launches_per_step"])' 2>&1 | tail -1)" >> gpurun_out/rv_n1.txt
}
for rep in 1 2 3; do
  one HP_X=head
  one HP_LIB_VARIANT=prefin
done
timeout 600 python bench.py --workload c3 --steps 20 --no-cpu-baseline --no-e2e > /tmp/c3.json 2>/dev/null
python -c 'import json; d=json.loads(open("/tmp/c3.json").read().strip().splitlines()[-1]); a=d["roofline"]["attention"]; print("C3", round(d["value"]), "attn replay", round(a["replay_ms_per_step"],4))' >> gpurun_out/rv_n1.txt
