#!/bin/bash
# quick GPU check: sanitizer on a tiny case, gpu tests, short bench
set -x
cd "$GRAFT_REPO_ROOT"
timeout 300 compute-sanitizer --tool memcheck python -c "
import sys; sys.path.insert(0,'.')
import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck.log 2>&1; tail -5 gpurun_out/memcheck.log
timeout 1500 python -m pytest tests -m gpu -q -x "$@" > gpurun_out/pytest_gpu.log 2>&1; tail -40 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-budget 8 > gpurun_out/bench.log 2>&1; tail -3 gpurun_out/bench.log
