#!/bin/bash
export HP_LIB_VARIANT=prof
for g in stream graph; do
  echo "== wo 4096x768x768 $g"; python tools/gemm_gap.py 4096 768 768 0 6 $g
  echo "== ffn1 4096x3072x768 $g"; python tools/gemm_gap.py 4096 3072 768 0 6 $g
  echo "== ffn1 nothing 4096x3072x768 $g"; python tools/gemm_gap.py 4096 3072 768 700000 6 $g
done
