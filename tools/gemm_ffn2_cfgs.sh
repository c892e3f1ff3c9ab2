#!/bin/bash
# the N = 768, K = 3072 projection under each tile config: full / no loads / MMA only
export HP_LIB_VARIANT=prof
for cfg in 1192 1256 2256 2128; do
  for d in 0 1 5; do
    echo "=== cfg $cfg debug $d"
    python tools/gemm_trace.py 4096 768 3072 $((d * 100000 + cfg)) | grep -E "CTAs|^tile|prologue"
  done
done
python tools/gemm_bench.py --only ffn2_fwd,dX1 --bn 2256
python tools/gemm_bench.py --only ffn2_fwd,dX1 --bn 1256
python tools/gemm_bench.py --only ffn2_fwd,dX1 --bn 1192
