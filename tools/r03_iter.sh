#!/bin/bash
# One optimisation iteration on a B200: fused-lattice parity tests (incl. virtual ranks / chunked
# exchange), then config-4 per-kernel event times for the given L1 cluster sizes.
set -u
timeout 900 python -m pytest tests/test_gpu_lattice_fused.py -m gpu -q -x 2>&1 | tail -3
for k in ${@:-4}; do echo "K=$k"; FMTGP_LAT_CLUSTER=$k timeout 300 python tools/prof_config4.py 5 --profile 2>&1 | tail -4; done
