#!/bin/bash
# final HEAD check on one GPU: smoke, the -m gpu suite, bench N=1, reference arm, then the ncu launch list of a short bench
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo EXIT $? >> gpurun_out/f_smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/f_tests.log 2>&1; echo EXIT $? >> gpurun_out/f_tests.log
timeout 400 python bench.py > gpurun_out/f_bench_n1.json 2> gpurun_out/f_bench_n1.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_ref_n1.json 2> gpurun_out/f_ref_n1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_ncu.log 2>&1; echo EXIT $? >> gpurun_out/f_ncu.log
