#!/bin/bash
# ncu --set full captures of the C2 step's kernels (one GPU): GEMMs, then attention / LN / Adam
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncu_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 150 -c 10 -o gpurun_out/r01c_gemm $CMD > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"attn_|adam_kernel|ln_bwd_bulk|ln_fwd_bulk" -s 80 -c 8 -o gpurun_out/r01c_mem $CMD > gpurun_out/ncu_mem.log 2>&1
