#!/bin/bash
# Round-2 final evidence on one GPU: smoke, the -m gpu suite, bench N=1 (C2),
# reference arm, C3 / C4 lines, ncu launch lists (cold + warm, DRAM bytes) and
# one ncu --set full capture of step GEMMs + attention
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo EXIT $? >> gpurun_out/g_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/g_tests.log 2>&1; echo EXIT $? >> gpurun_out/g_tests.log
timeout 400 python bench.py > gpurun_out/g_bench_n1.json 2> gpurun_out/g_bench_n1.err
timeout 400 python bench.py --impl reference > gpurun_out/g_ref_n1.json 2> gpurun_out/g_ref_n1.err
timeout 400 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/g_bench_c3.json 2> gpurun_out/g_bench_c3.err
timeout 600 python bench.py --workload c4 --steps 10 --no-cpu-baseline > gpurun_out/g_bench_c4.json 2> gpurun_out/g_bench_c4.err
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-same-config --no-loss-check"
timeout 600 $CMD > gpurun_out/g_plain.json 2> gpurun_out/g_plain.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 900 -c 860 --csv --log-file gpurun_out/g_launches_cold.csv $CMD > gpurun_out/g_ncu_cold.log 2>&1; echo EXIT $? >> gpurun_out/g_ncu_cold.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -s 900 -c 860 --csv --log-file gpurun_out/g_launches_warm.csv $CMD > gpurun_out/g_ncu_warm.log 2>&1; echo EXIT $? >> gpurun_out/g_ncu_warm.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc_kernel|attn_" -s 950 -c 8 -o gpurun_out/g_full $CMD > gpurun_out/g_ncu_full.log 2>&1; echo EXIT $? >> gpurun_out/g_ncu_full.log
