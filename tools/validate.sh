#!/bin/bash
# GPU validation: the full -m gpu suite (2 GPUs -> multi-GPU tests run), bench at N=1 and N=2
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/v_tests.log 2>&1; echo EXIT $? >> gpurun_out/v_tests.log
timeout 300 python bench.py > gpurun_out/v_bench_n1.json 2> gpurun_out/v_bench_n1.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 > gpurun_out/v_bench_n2.json 2> gpurun_out/v_bench_n2.err
