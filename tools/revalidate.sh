#!/bin/bash
# HEAD re-validation on one GPU after a container rebuild: smoke, the -m gpu suite, bench N=1, reference arm
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo EXIT $? >> gpurun_out/v_smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/v_tests.log 2>&1; echo EXIT $? >> gpurun_out/v_tests.log
timeout 400 python bench.py > gpurun_out/v_bench_n1.json 2> gpurun_out/v_bench_n1.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v_ref_n1.json 2> gpurun_out/v_ref_n1.err
