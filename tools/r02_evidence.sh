#!/bin/bash
# Round-2 evidence on one B200: parity suite, smoke, bench lines (config 4 default + reference arm,
# configs 1/2/3/5), launch list of the default bench command, ncu --set full of the three fused
# lattice kernels (CSV exports only; the report stays in /tmp).
set -u
mkdir -p gpurun_out
tag=${1:-r02}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; tail -2 gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; tail -1 gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench_c4.log 2>&1; tail -1 gpurun_out/${tag}_bench_c4.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_ref.log 2>&1; tail -1 gpurun_out/${tag}_bench_ref.log | cut -c1-200
for c in 1 2 3 5; do
  st=20; [ $c = 3 ] && st=3; [ $c = 5 ] && st=5
  timeout 900 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/${tag}_bench_c$c.log 2>&1; tail -1 gpurun_out/${tag}_bench_c$c.log | cut -c1-200
done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_lat_(col|mid)" -c 3 -f -o /tmp/${tag}_c4full \
      python tools/prof_config4.py 1 > gpurun_out/${tag}_ncu_c4.log 2>&1; tail -1 gpurun_out/${tag}_ncu_c4.log
ncu -i /tmp/${tag}_c4full.ncu-rep --page raw --csv > gpurun_out/${tag}_ncu_full_config4_raw.csv 2>/dev/null
ls -la gpurun_out | tail -20
