#!/bin/bash
# A/B of library builds on one B200 in one call: config-4 per-kernel event times for the given
# libraries (FMTGP_LIB override; default ab/*.so), twice each, interleaved.  TEST=lib first runs the
# fused-lattice parity tests against that library.
set -u
libs=${@:-ab/*.so}
if [ -n "${TEST:-}" ]; then
  for t in $TEST; do echo "== tests with $t"; FMTGP_LIB=$PWD/$t timeout 900 python -m pytest tests/test_gpu_lattice_fused.py tests/test_gpu_baseline_shapes.py -m gpu -q -x 2>&1 | tail -3; done
fi
for rep in 1 2; do
  for lib in $libs; do
    echo "== $lib"
    FMTGP_LIB=$PWD/$lib timeout 300 python tools/prof_config4.py 5 --profile 2>&1 | tail -4 | tr '\n' ' '; echo
  done
done
