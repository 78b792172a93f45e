#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 300 python tools/prof_config4.py 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_lat_(mid|col_inv)" -c 2 -f -o /tmp/c4m python tools/prof_config4.py 1 > /dev/null 2>&1
ncu -i /tmp/c4m.ncu-rep -k regex:k_lat_mid --page source --csv --print-source sass > gpurun_out/r02d_sass_mid.csv 2>/dev/null
ncu -i /tmp/c4m.ncu-rep -k regex:k_lat_col_inv --page source --csv --print-source sass > gpurun_out/r02d_sass_inv.csv 2>/dev/null
ls -la gpurun_out
