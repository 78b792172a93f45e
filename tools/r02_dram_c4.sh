#!/bin/bash
# config-4 lattice kernels: DRAM bytes + time per kernel, L2 prefetch variants (FMTGP_LAT_PF)
set -u
mkdir -p gpurun_out
timeout 300 python tools/prof_config4.py 3 > gpurun_out/dram_prof.log 2>&1; tail -1 gpurun_out/dram_prof.log
for pf in 0 1; do
  FMTGP_LAT_PF=$pf timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control none -k regex:"k_lat_(col|mid)" -c 3 --csv python tools/prof_config4.py 1 > gpurun_out/dram_pf$pf.csv 2>gpurun_out/dram_pf$pf.err
  echo "pf=$pf"; grep -E "k_lat" gpurun_out/dram_pf$pf.csv | awk -F'","' '{print $5" | "$(NF-2)" "$(NF-1)" "$NF}' | cut -c1-200
done
