#!/bin/bash
# A/B: two ring slots per producer / MMA loop iteration (default) vs one (kb1)
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm or x6" > gpurun_out/abkb_tests.log 2>&1; echo EXIT $? >> gpurun_out/abkb_tests.log
python tools/gemm_bench.py > gpurun_out/abkb_gemm_kb2.txt 2>&1
HP_LIB_VARIANT=kb1 python tools/gemm_bench.py > gpurun_out/abkb_gemm_kb1.txt 2>&1
export HP_LIB_VARIANT=prof
for cfg in 1128 1192 2128 2256; do
  for d in 5 0; do
    echo "=== cfg $cfg debug $d" >> gpurun_out/abkb_trace.txt
    python tools/gemm_trace.py 4096 3072 3072 $((d * 100000 + cfg)) | grep -E "CTAs|^tile" >> gpurun_out/abkb_trace.txt
  done
done
unset HP_LIB_VARIANT
one() {
  env "$@" timeout 300 python bench.py --steps 40 --no-cpu-baseline --no-e2e --no-same-config > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["value"]), round(d["ms_per_step"],4), round(r["gemm_ms_per_step"],4), round(r["frac"],4))' 2>&1 | tail -1)" >> gpurun_out/abkb.txt
}
for rep in 1 2 3; do
  one HP_X=base
  one HP_LIB_VARIANT=kb1
done
