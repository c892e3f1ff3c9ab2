#!/bin/bash
# A/B: GEMM epilogue C / aux via TMA store from the staging tile (new) vs st.global (base)
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm or x6" > gpurun_out/abt_tests.log 2>&1; echo EXIT $? >> gpurun_out/abt_tests.log
python tools/gemm_bench.py > gpurun_out/abt_gemm_new.txt 2>&1
HP_GEMM_TMA_STORE=0 python tools/gemm_bench.py > gpurun_out/abt_gemm_off.txt 2>&1
python tools/gemm_bench.py --only variants > gpurun_out/abt_var_new.txt 2>&1
HP_GEMM_TMA_STORE=0 python tools/gemm_bench.py --only variants > gpurun_out/abt_var_off.txt 2>&1
one() {
  env "$@" timeout 300 python bench.py --steps 40 --no-cpu-baseline --no-e2e --no-same-config > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["value"]), round(d["ms_per_step"],4), round(r["replay"]["ms_per_step"],4), round(r["frac"],4))' 2>&1 | tail -1)" >> gpurun_out/abt.txt
}
for rep in 1 2 3; do
  one HP_X=new
  one HP_GEMM_TMA_STORE=0
done
