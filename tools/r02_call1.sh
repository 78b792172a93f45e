#!/bin/bash
# round-2 first GPU call: parity suite, default bench (config 4), fp64 roof, reference scaling check
set -u
mkdir -p gpurun_out
./tools/micro/fp64_peak > gpurun_out/r02_fp64_peak.log 2>&1; cat gpurun_out/r02_fp64_peak.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_gpu.log 2>&1; tail -15 gpurun_out/r02_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r02_bench_c4.log 2>&1; tail -1 gpurun_out/r02_bench_c4.log | cut -c1-600
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/r02_bench_c2.log 2>&1; tail -1 gpurun_out/r02_bench_c2.log | cut -c1-300
timeout 900 python tools/ref_scaling.py --max-m 26 > gpurun_out/r02_ref_scaling.json 2> gpurun_out/r02_ref_scaling.err; tail -3 gpurun_out/r02_ref_scaling.err
