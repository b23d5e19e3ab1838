#!/bin/bash
# quick NN iteration: NN parity tests, bench NN phases (C2 + north_star C4), clock-probe phase split
cd "$GRAFT_REPO_ROOT"
R=${1:-q}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "nn" > gpurun_out/nn_tests_$R.log 2>&1; tail -1 gpurun_out/nn_tests_$R.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --compare "" --no-two-stage > gpurun_out/bench_$R.log 2>&1
tail -1 gpurun_out/bench_$R.log | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); c=d.get('north_star_c4',{})
  print(round(d['value']), d['phase_ms_per_step'], round(c.get('value',0)), c.get('phase_ms_per_step'))
except Exception as e: print('ERR', e)"
python scripts/nn_phases.py --config C2 --M 10000; python scripts/nn_phases.py --config C4 --M 65536
