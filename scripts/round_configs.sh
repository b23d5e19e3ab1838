#!/bin/bash
# Full-size configs C1-C4 (sampled parity) and the C5 sweep with the current build.
# usage: bash scripts/round_configs.sh rNN
R=${1:-r01}
cd "$GRAFT_REPO_ROOT"
for c in C1 C2 C3 C3j C4; do
  timeout 900 python scripts/run_config.py --config $c --form incremental --out gpurun_out/cfg_${c}_$R.json \
      > gpurun_out/cfg_${c}_$R.log 2>&1; tail -c 400 gpurun_out/cfg_${c}_$R.log; echo
done
timeout 1800 python scripts/c5_sweep.py --out gpurun_out/c5_sweep_$R.jsonl > gpurun_out/c5_$R.log 2>&1; tail -2 gpurun_out/c5_$R.log
