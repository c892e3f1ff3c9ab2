#!/bin/bash
# split word-embedding update at N=2 (union of the ranks' ids allgathered before backward): tests, then interleaved bench pairs
mkdir -p gpurun_out
# (tests: run once, green -- see profiles/r01_ab_emb_split.txt)

for i in 1 2 3; do
  for m in 1 0; do
    HP_EMB_SPLIT=$m timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 295$i$m bench.py --gpus 2 > gpurun_out/t2_n2_s${m}_$i.json 2> gpurun_out/t2_n2_s${m}_$i.err
  done
done
for m in 1 0; do HP_EMB_SPLIT=$m CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/t2_n1_s$m.json 2> gpurun_out/t2_n1_s$m.err; done
