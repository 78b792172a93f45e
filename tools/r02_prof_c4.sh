#!/bin/bash
# config-4 lattice kernels: one ncu --set full capture with source (after a clean run)
set -u
mkdir -p gpurun_out
timeout 300 python tools/prof_config4.py 3 --profile > gpurun_out/r02_prof_c4.log 2>&1; cat gpurun_out/r02_prof_c4.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_lat -c 3 -f -o gpurun_out/r02_c4 python tools/prof_config4.py 1 > gpurun_out/r02_c4_ncu.log 2>&1; tail -3 gpurun_out/r02_c4_ncu.log
