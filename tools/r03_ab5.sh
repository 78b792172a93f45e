#!/bin/bash
# A/B of library builds on config 5 (256-candidate sweep) and config 2: tools/r03_ab5.sh lib1 lib2 ...
set -u
if [ -n "${TEST:-}" ]; then
  for t in $TEST; do echo "== tests with $t"; FMTGP_LIB=$PWD/$t timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_shapes.py tests/test_gpu_digital_sweep.py -m gpu -q -x 2>&1 | tail -3; done
fi
for rep in 1 2; do
  for lib in $@; do
    echo "== $lib"
    FMTGP_LIB=$PWD/$lib timeout 300 python tools/prof_config5.py 4 --profile 2>&1 | tail -6 | tr '\n' ' '; echo
    FMTGP_LIB=$PWD/$lib timeout 300 python bench.py --config 2 --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  config2', round(d['value'],1), 'fits/s', d['ms_per_step'])"
  done
done
