#!/bin/bash
# Where a tcgen05 GEMM's time goes: the HP_GEMM_PROFILE build's debug bits
# (1 = no TMA loads, MMA on stale smem; 2 = no MMA; 4 = no epilogue work)
# on the C2 shapes, graph-replayed (tools/gemm_bench.py --bn debug*100000)
export HP_LIB_VARIANT=prof
S=ffn1_fwd_gelu,ffn2_fwd,dW2,wo_fwd,dX1,dU_dgelu,v_plain_bf16
for d in 0 1 4 5 2 3 6; do
  echo "== debug $d"
  python tools/gemm_bench.py --only $S --bn $((d * 100000)) --iters 20 | grep -v "step GEMM"
done
