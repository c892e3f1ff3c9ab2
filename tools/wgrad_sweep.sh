#!/bin/bash
# weight-gradient GEMM configurations: code = splits*10000 + cg*1000 + bn (splits 0 = heuristic)
for code in 0 12256 22256 42256 12128 22128 11128 21128 41128 11256 21256 11192 21192; do
  echo "== code $code"; timeout 60 python tools/gemm_bench.py --iters 20 --only dW2,dW1,dWo,dWqkv --bn $code | grep -v "step GEMM"
done
