#!/bin/bash
# HEAD validation on two GPUs: smoke, the -m gpu suite (multi-GPU tests included), bench N=1 and N=2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo EXIT $? >> gpurun_out/g_smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g_tests.log 2>&1; echo EXIT $? >> gpurun_out/g_tests.log
timeout 400 python bench.py > gpurun_out/g_bench_n1.json 2> gpurun_out/g_bench_n1.err
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 > gpurun_out/g_bench_n2.json 2> gpurun_out/g_bench_n2.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/g_ref_n2.json 2> gpurun_out/g_ref_n2.err
