#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v2_tests.log 2>&1; echo EXIT $? >> gpurun_out/v2_tests.log
for i in 1 2; do timeout 300 python bench.py > gpurun_out/v2_bench_n1_$i.json 2> gpurun_out/v2_bench_n1_$i.err; done
