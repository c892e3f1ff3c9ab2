#!/bin/bash
# MMA-only rate per (CTA group, N tile): debug bits 1+4 (no loads, no epilogue),
# tile-to-tile epilogue-start spacing from tools/gemm_trace.py (CTA 0, cycles)
export HP_LIB_VARIANT=prof
for cfg in 1128 1192 1256 2128 2256; do
  for d in 5 1 0; do
    echo "=== cfg $cfg debug $d"
    python tools/gemm_trace.py 4096 3072 3072 $((d * 100000 + cfg)) | grep -E "CTAs|^tile|prologue"
  done
done
