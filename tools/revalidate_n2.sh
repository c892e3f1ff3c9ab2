#!/bin/bash
# HEAD on two GPUs: the multi-GPU tests, bench N=1 and N=2 back to back, reference arm at N=2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/m_tests.log 2>&1; echo EXIT $? >> gpurun_out/m_tests.log
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > gpurun_out/m_bench_n1.json 2> gpurun_out/m_bench_n1.err
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 > gpurun_out/m_bench_n2.json 2> gpurun_out/m_bench_n2.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29572 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/m_ref_n2.json 2> gpurun_out/m_ref_n2.err
