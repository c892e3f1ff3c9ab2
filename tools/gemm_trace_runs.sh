#!/bin/bash
# CTA timelines (tools/gemm_trace.py) of the N = 768 / K = 768 C2 GEMMs, normal and
# with debug bits (1 no loads, 2 no MMA, 4 no epilogue), HP_GEMM_PROFILE build
export HP_LIB_VARIANT=prof
for code in 0 300000 500000 700000; do
  echo "=== wo_fwd 4096x768x768 code $code"; python tools/gemm_trace.py 4096 768 768 $code
  echo "=== ffn2 4096x768x3072 code $code"; python tools/gemm_trace.py 4096 768 3072 $code
done
echo "=== v_plain 4096x3072x768 code 0"; python tools/gemm_trace.py 4096 3072 768 0
echo "=== v_plain 4096x3072x768 code 500000"; python tools/gemm_trace.py 4096 3072 768 500000
