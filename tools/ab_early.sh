#!/bin/bash
# A/B: first ring slots loaded before the CTA / cluster barrier (new) vs after (base = previous HEAD)
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm or x6" > gpurun_out/abe_tests.log 2>&1; echo EXIT $? >> gpurun_out/abe_tests.log
python tools/gemm_bench.py > gpurun_out/abe_gemm_new.txt 2>&1
HP_LIB_VARIANT=base python tools/gemm_bench.py > gpurun_out/abe_gemm_base.txt 2>&1
HP_LIB_VARIANT=prof python tools/gemm_trace.py 4096 768 768 0 > gpurun_out/abe_trace_wo.txt 2>&1
HP_LIB_VARIANT=prof python tools/gemm_trace.py 4096 3072 768 0 > gpurun_out/abe_trace_ffn1.txt 2>&1
one() {
  env "$@" timeout 300 python bench.py --steps 40 --no-cpu-baseline --no-e2e --no-same-config > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["value"]), round(d["ms_per_step"],4), round(r["replay"]["ms_per_step"],4), round(r["frac"],4))' 2>&1 | tail -1)" >> gpurun_out/abe.txt
}
for rep in 1 2 3; do
  one HP_X=new
  one HP_LIB_VARIANT=base
done
