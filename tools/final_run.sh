#!/bin/bash
# Round evidence on one GPU: smoke, the -m gpu suite, bench (default), reference arm, warm launch list
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo EXIT $? >> gpurun_out/f_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f_tests.log 2>&1; echo EXIT $? >> gpurun_out/f_tests.log
timeout 400 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_ref.json 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_ncu.log 2>&1
