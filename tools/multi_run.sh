set -x
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/m_bench_n1.json 2> gpurun_out/m_bench_n1.err
for N in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 30 --warmup 5 > gpurun_out/m_bench_n$N.json 2> gpurun_out/m_bench_n$N.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N tools/allreduce_sweep.py > gpurun_out/m_sweep_n$N.json 2> gpurun_out/m_sweep_n$N.err
done
