#!/bin/bash
# bf16x6 fp32 GEMMs: all K-chunk partials in one launch (new) -- full GPU suite + bench same_config
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/abs_tests.log 2>&1; echo EXIT $? >> gpurun_out/abs_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/abs_bench.json 2> gpurun_out/abs_bench.err
HP_LIB_VARIANT=base timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/abs_bench_base.json 2> gpurun_out/abs_bench_base.err
