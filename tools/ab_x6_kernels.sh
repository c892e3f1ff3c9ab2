#!/bin/bash
# bf16x6 helpers: vectorised partial reduction, paired split6 stores -- GPU suite, same_config, f32 launch list
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/abrs_tests.log 2>&1; echo EXIT $? >> gpurun_out/abrs_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/abrs_bench.json 2> gpurun_out/abrs_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/abrs_f32_launches.csv python tools/f32_profile.py 1 > gpurun_out/abrs_ncu.log 2>&1; echo EXIT $? >> gpurun_out/abrs_ncu.log
