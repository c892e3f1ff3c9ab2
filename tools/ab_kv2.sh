#!/bin/bash
# C4 long attention: dK/dV kernel at two CTAs per SM (attn_bwd_kv_long2, default) vs one (HP_ATTN_LONG_KV2=0)
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_bench_shapes.py -x -q -k "long or c4" > gpurun_out/abk_tests.log 2>&1; echo EXIT $? >> gpurun_out/abk_tests.log
one() {
  env "$@" timeout 600 python bench.py --workload c4 --steps 10 --no-cpu-baseline --no-e2e --no-same-config --no-loss-check > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); r=d["roofline"]; a=r["attention"]; print(round(d["value"],1), round(d["ms_per_step"],3), "attn replay", round(a["replay_ms_per_step"],3), "in-step", round(a["ms_per_step"],3))' 2>&1 | tail -1)" >> gpurun_out/abk.txt
}
for rep in 1 2; do
  one HP_X=kv2
  one HP_ATTN_LONG_KV2=0
done
CMD="python bench.py --workload c4 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline --no-same-config --no-loss-check"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_ --csv --log-file gpurun_out/abk_launches.csv $CMD > gpurun_out/abk_ncu.log 2>&1; echo EXIT $? >> gpurun_out/abk_ncu.log
