#!/bin/bash
# config-4 lattice kernels: one ncu --set full capture with source (after a clean run)
set -u
mkdir -p gpurun_out
tag=${1:-r02_c4}
timeout 300 python tools/prof_config4.py 3 --profile > gpurun_out/${tag}_prof.log 2>&1; cat gpurun_out/${tag}_prof.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_lat_[cm] -c 3 -f -o gpurun_out/${tag} python tools/prof_config4.py 1 > gpurun_out/${tag}_ncu.log 2>&1; tail -2 gpurun_out/${tag}_ncu.log
