#!/bin/bash
# Round-2 evidence on one B200: parity suite, smoke, bench (config 4 default) + reference arm,
# launch list of the bench command, ncu --set full of the three fused lattice kernels.
set -u
mkdir -p gpurun_out
tag=${1:-r02}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; tail -2 gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; tail -1 gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench_c4.log 2>&1; tail -1 gpurun_out/${tag}_bench_c4.log | cut -c1-400
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_ref.log 2>&1; tail -1 gpurun_out/${tag}_bench_ref.log | cut -c1-300
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/${tag}_bench_c2.log 2>&1; tail -1 gpurun_out/${tag}_bench_c2.log | cut -c1-200
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_c5.log 2>&1; tail -1 gpurun_out/${tag}_bench_c5.log | cut -c1-200
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_lat_(col|mid)" -c 3 -f -o gpurun_out/${tag}_c4full \
      python tools/prof_config4.py 1 > gpurun_out/${tag}_ncu_c4.log 2>&1; tail -1 gpurun_out/${tag}_ncu_c4.log
