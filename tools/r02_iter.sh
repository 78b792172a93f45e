#!/bin/bash
# quick iteration: fused-lattice parity tests + config-4 kernel timings
set -u
timeout 600 python -m pytest tests/test_gpu_lattice_fused.py tests/test_gpu_baseline_shapes.py -m gpu -q -x 2>&1 | tail -3
timeout 300 python tools/prof_config4.py 3 --profile 2>&1 | tail -4
