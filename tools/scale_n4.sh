#!/bin/bash
# HEAD scaling on one 4-GPU box: bench N=1, 2, 4 back to back (C2, driver defaults)
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > gpurun_out/q_n1.json 2> gpurun_out/q_n1.err
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus 2 > gpurun_out/q_n2.json 2> gpurun_out/q_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29592 bench.py --gpus 4 > gpurun_out/q_n4.json 2> gpurun_out/q_n4.err
