#!/bin/bash
# SASS-level capture of the three fused lattice kernels (config 4): per-opcode executed counts,
# stalls, top SASS lines and top CUDA lines.  bash tools/r03_sass_c4.sh TAG
set -u
mkdir -p gpurun_out
tag=${1:-r03}
timeout 300 python tools/prof_config4.py 3 --profile || exit 1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_lat_(col|mid)" -c 3 -f -o /tmp/${tag}_c4 python tools/prof_config4.py 1 > gpurun_out/${tag}_ncu.log 2>&1
for k in k_lat_col_fwd k_lat_mid k_lat_col_inv; do
  ncu -i /tmp/${tag}_c4.ncu-rep -k regex:$k --page source --csv --print-source sass > /tmp/${tag}_$k.csv 2>/dev/null
  ncu -i /tmp/${tag}_c4.ncu-rep -k regex:$k --page source --csv --print-source cuda,sass > /tmp/${tag}_${k}_cs.csv 2>/dev/null
  python tools/ncu_sass_stats.py /tmp/${tag}_${k}_cs.csv > gpurun_out/${tag}_sass_stats_$k.txt 2>&1
  python tools/ncu_sass_top.py /tmp/${tag}_$k.csv > gpurun_out/${tag}_sass_top_$k.txt 2>&1
  python tools/ncu_src_top.py /tmp/${tag}_${k}_cs.csv 40 > gpurun_out/${tag}_src_top_$k.txt 2>&1
  gzip -c /tmp/${tag}_${k}_cs.csv > gpurun_out/${tag}_${k}_cs.csv.gz
done
ncu -i /tmp/${tag}_c4.ncu-rep --page raw --csv > gpurun_out/${tag}_ncu_full_config4_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/${tag}_ncu_full_config4_raw.csv > gpurun_out/${tag}_config4_ncu_summary.txt 2>&1
