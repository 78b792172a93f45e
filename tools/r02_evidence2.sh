#!/bin/bash
# Round-2 evidence, part 2: config 1 / 5 bench lines, config-5 kernels under ncu --set full
set -u
mkdir -p gpurun_out
tag=${1:-r02b}
timeout 600 python bench.py --config 1 --no-cpu-baseline > gpurun_out/${tag}_bench_c1.log 2>&1; tail -1 gpurun_out/${tag}_bench_c1.log | cut -c1-300
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/${tag}_bench_c5.log 2>&1; tail -1 gpurun_out/${tag}_bench_c5.log | cut -c1-300
timeout 300 python tools/prof_config5.py 3 64 --profile > gpurun_out/${tag}_prof_c5.log 2>&1; tail -6 gpurun_out/${tag}_prof_c5.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_dig_(col|mid)" -s 3 -c 3 -f -o gpurun_out/${tag}_c5full \
      python tools/prof_config5.py 1 64 > gpurun_out/${tag}_ncu_c5.log 2>&1; tail -1 gpurun_out/${tag}_ncu_c5.log
