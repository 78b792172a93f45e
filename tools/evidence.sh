#!/bin/bash
# Round evidence on one B200 (run via gpurun): parity suite, bench lines (config 2 default, config 4),
# launch list of the bench command, ncu --set full of the config-2 and config-4 kernels, full-size
# config runs.  Outputs in gpurun_out/ (ncu reports stay in /tmp: only their CSV exports travel).
set -u
python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.log 2>&1; tail -2 gpurun_out/ev_pytest_gpu.log
python bench.py > gpurun_out/ev_bench.log 2>&1; tail -1 gpurun_out/ev_bench.log | cut -c1-400
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev_bench_ref.log 2>&1; tail -1 gpurun_out/ev_bench_ref.log | cut -c1-300
python bench.py --config 4 --steps 5 --warmup 3 > gpurun_out/ev_bench_c4.log 2>&1; tail -1 gpurun_out/ev_bench_c4.log | cut -c1-300
python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/ev_bench_c5.log 2>&1; tail -1 gpurun_out/ev_bench_c5.log | cut -c1-300
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; tail -1 gpurun_out/ev_smoke.log
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev_bench_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_launch.log 2>&1
python tools/prof_config2.py 3 > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:"k_dig_(col|mid)" -s 3 -c 3 -f -o /tmp/ev_c2 \
      python tools/prof_config2.py 3 > gpurun_out/ev_ncu_full.log 2>&1
ncu -i /tmp/ev_c2.ncu-rep --page raw --csv > gpurun_out/ev_ncu_full_raw.csv 2>/dev/null
python tools/prof_config4.py 1 > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:"k_lat" -c 3 -f -o /tmp/ev_c4 \
      python tools/prof_config4.py 1 > gpurun_out/ev_ncu_c4.log 2>&1
ncu -i /tmp/ev_c4.ncu-rep --page raw --csv > gpurun_out/ev_ncu_c4_raw.csv 2>/dev/null
python tools/prof_config5.py 3 --profile > gpurun_out/ev_config5.log 2>&1; tail -5 gpurun_out/ev_config5.log
python tools/trace_config2.py 3 > gpurun_out/ev_trace_c2.log 2>&1
python tools/run_configs.py --configs 1,2,3,4,5 > gpurun_out/ev_configs.log 2>&1; tail -5 gpurun_out/ev_configs.log | cut -c1-200
