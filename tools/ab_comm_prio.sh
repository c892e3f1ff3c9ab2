#!/bin/bash
# NCCL bucket stream priority A/B at N=4 and N=2 (HP_COMM_PRIO=hi vs the default low priority), interleaved
mkdir -p gpurun_out
for i in 1 2 3; do
  for m in hi lo; do
    HP_COMM_PRIO=$m timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 296$i${#m} bench.py --gpus 4 --no-e2e > gpurun_out/p4_${m}_$i.json 2> gpurun_out/p4_${m}_$i.err
  done
done
for i in 1 2; do
  for m in hi lo; do
    HP_COMM_PRIO=$m CUDA_VISIBLE_DEVICES=0,1 timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 297$i${#m} bench.py --gpus 2 --no-e2e > gpurun_out/p2_${m}_$i.json 2> gpurun_out/p2_${m}_$i.err
  done
done
