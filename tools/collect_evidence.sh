#!/bin/bash
# Copies one evidence call's outputs (gpurun_out/TAG_*) into profiles/ under the round's names.
# tools/collect_evidence.sh TAG [ROUND]   e.g.  tools/collect_evidence.sh r03b r02
set -eu
tag=$1; rnd=${2:-r02}
cd "$(dirname "$0")/.."
for c in c1 c2 c3 c4 c5 ref; do
  f=gpurun_out/${tag}_bench_$c.log
  [ -f $f ] && tail -1 $f > profiles/${rnd}_bench_$c.json
done
[ -f gpurun_out/${tag}_launches.csv ] && cp gpurun_out/${tag}_launches.csv profiles/${rnd}_launches_config4.csv
if [ -f gpurun_out/${tag}_ncu_full_config4_raw.csv ]; then
  cp gpurun_out/${tag}_ncu_full_config4_raw.csv profiles/${rnd}_ncu_full_config4_raw.csv
  python tools/ncu_summary.py profiles/${rnd}_ncu_full_config4_raw.csv > profiles/${rnd}_config4_ncu_summary.txt
fi
[ -f gpurun_out/${tag}_pytest_gpu.log ] && cp gpurun_out/${tag}_pytest_gpu.log profiles/${rnd}_pytest_gpu.log
[ -f gpurun_out/${tag}_smoke.log ] && cp gpurun_out/${tag}_smoke.log profiles/${rnd}_smoke.log
ls -la profiles | grep ${rnd}_ | head -30
