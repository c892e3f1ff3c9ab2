#!/bin/bash
python tools/gemm_bench.py > gpurun_out/abfs_gemm_new.txt 2>&1
HP_LIB_VARIANT=base python tools/gemm_bench.py > gpurun_out/abfs_gemm_base.txt 2>&1
for sp in 1 2 3 4; do
  echo "== 2256 splits $sp" >> gpurun_out/abfs_gemm_forced.txt
  python tools/gemm_bench.py --only ffn2_fwd,dX1,dX,wo_fwd,dW2,dW1,dWo --bn $((2256 + 10000 * sp)) | grep -v step >> gpurun_out/abfs_gemm_forced.txt 2>&1
done
