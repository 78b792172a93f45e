#!/bin/bash
# config-5 kernels under ncu --set full; exports only (the report itself stays in /tmp)
set -u
mkdir -p gpurun_out
timeout 300 python tools/prof_config5.py 1 64 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_dig_(col|mid)" -s 3 -c 3 -f -o /tmp/c5full \
      python tools/prof_config5.py 1 64 > gpurun_out/r03e_ncu_c5.log 2>&1; tail -1 gpurun_out/r03e_ncu_c5.log
ncu -i /tmp/c5full.ncu-rep --page raw --csv > gpurun_out/r03e_ncu_full_config5_raw.csv 2>/dev/null
for k in col_fwd mid col_inv; do ncu -i /tmp/c5full.ncu-rep -k regex:k_dig_$k --page source --csv --print-source sass > gpurun_out/r03e_sass_c5_$k.csv 2>/dev/null; done
ls -la gpurun_out/
