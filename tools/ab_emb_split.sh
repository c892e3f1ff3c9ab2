#!/bin/bash
# split word-embedding update (adam_rows) vs the dense last-bucket update: GPU tests, then interleaved N=1 bench pairs
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_engine.py -x -q -k split > gpurun_out/s_split_test.log 2>&1; echo EXIT $? >> gpurun_out/s_split_test.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s_tests.log 2>&1; echo EXIT $? >> gpurun_out/s_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s_smoke.log 2>&1; echo EXIT $? >> gpurun_out/s_smoke.log
for i in 1 2 3; do
  HP_EMB_SPLIT=1 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/s_split_$i.json 2>gpurun_out/s_split_$i.err
  HP_EMB_SPLIT=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/s_dense_$i.json 2>gpurun_out/s_dense_$i.err
done
