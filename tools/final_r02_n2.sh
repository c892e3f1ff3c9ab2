#!/bin/bash
# Round-2 final evidence on a 2-GPU box: the multi-GPU tests (skipped on one
# GPU) and bench N=1 / N=2 back to back (+ the reference arm at N=2)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -k "multi or w2 or two or nccl or comm" > gpurun_out/h_tests_2gpu.log 2>&1; echo EXIT $? >> gpurun_out/h_tests_2gpu.log
timeout 400 python bench.py > gpurun_out/h_bench_n1.json 2> gpurun_out/h_bench_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 2 > gpurun_out/h_bench_n2.json 2> gpurun_out/h_bench_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 bench.py --impl reference --gpus 2 > gpurun_out/h_ref_n2.json 2> gpurun_out/h_ref_n2.err
