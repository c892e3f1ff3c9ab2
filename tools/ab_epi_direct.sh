#!/bin/bash
# A/B: GEMM epilogue outputs straight from registers (each lane its own row's
# 64 / 128 B, no smem staging: "direct") vs TMA store from the staging tile
# (default of this build) vs st.global from the staging tile (TMA_STORE=0)
HP_LIB_VARIANT=direct timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm or x6" > gpurun_out/abx_tests.log 2>&1; echo EXIT $? >> gpurun_out/abx_tests.log
HP_LIB_VARIANT=direct python tools/gemm_bench.py > gpurun_out/abx_gemm_direct.txt 2>&1
python tools/gemm_bench.py > gpurun_out/abx_gemm_tma.txt 2>&1
HP_LIB_VARIANT=direct python tools/gemm_bench.py --only variants > gpurun_out/abx_var_direct.txt 2>&1
python tools/gemm_bench.py --only variants > gpurun_out/abx_var_tma.txt 2>&1
one() {
  env "$@" timeout 300 python bench.py --steps 40 --no-cpu-baseline --no-e2e --no-same-config > /tmp/o.json 2>/tmp/o.err
  echo "[$*] $(python -c 'import json,sys; d=json.loads(open("/tmp/o.json").read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["value"]), round(d["ms_per_step"],4), round(r["replay"]["ms_per_step"],4), round(r["frac"],4))' 2>&1 | tail -1)" >> gpurun_out/abx.txt
}
for rep in 1 2 3; do
  one HP_LIB_VARIANT=direct
  one HP_X=tma
  one HP_GEMM_TMA_STORE=0
done
