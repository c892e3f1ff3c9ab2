for code in 0 2128 12128 2256 12256 22256 1128 11128 21128 41128 1256 11256 21256; do
  echo "== code $code"; timeout 60 python tools/gemm_bench.py --iters 20 --only dW2,dW1,dWo,dWqkv --bn $code | grep -v "step GEMM"
done
