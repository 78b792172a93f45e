#!/bin/bash
set -u
timeout 600 python -m pytest tests/test_gpu_lattice_fused.py -m gpu -q -x 2>&1 | tail -3
for k in 1 2 4; do echo "K=$k"; FMTGP_LAT_CLUSTER=$k timeout 300 python tools/prof_config4.py 3 --profile 2>&1 | tail -4; done
