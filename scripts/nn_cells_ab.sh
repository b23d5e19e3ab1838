#!/bin/bash
# NN multi-axis cell grid: parity tests of the NN pool, then bench NN phase times
# (C2 and north_star C4) for the default grid, cell-size variants and the two-axis grid.
cd "$GRAFT_REPO_ROOT"
R=${1:-nnc}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "nn" > gpurun_out/nn_tests_$R.log 2>&1; tail -2 gpurun_out/nn_tests_$R.log
for v in "" "LAGP_NN_CR=128" "LAGP_NN_CR=512" "LAGP_NN_CELLS=2"; do
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --compare "" --no-two-stage > gpurun_out/bench_${R}_${v:-def}.log 2>&1
  echo "$v: $(tail -1 gpurun_out/bench_${R}_${v:-def}.log | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); c=d.get('north_star_c4',{})
  print(round(d['value']), d['phase_ms_per_step'], round(c.get('value',0)), c.get('phase_ms_per_step'))
except Exception as e: print('ERR', e)")"
done
