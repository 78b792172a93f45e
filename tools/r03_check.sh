#!/bin/bash
# Re-entry check on one B200: parity suite, smoke, default bench line, config-4 per-kernel times.
set -u
mkdir -p gpurun_out
tag=${1:-r02b}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; tail -2 gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; tail -1 gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench_c4.log 2>&1; tail -1 gpurun_out/${tag}_bench_c4.log | cut -c1-400
timeout 300 python tools/prof_config4.py 3 --profile 2>&1 | tail -6
