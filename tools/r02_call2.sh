#!/bin/bash
# round-2 status call: parity suite + default bench (config 4) + config 2 line
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_gpu.log 2>&1; tail -15 gpurun_out/r02_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02_bench_c4.log 2>&1; tail -1 gpurun_out/r02_bench_c4.log | cut -c1-1500
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/r02_bench_c2.log 2>&1; tail -1 gpurun_out/r02_bench_c2.log | cut -c1-600
