#!/bin/bash
# Round evidence: bench line, launch list, ncu full captures of the local-design
# kernels and the NN kernel at the bench's launch configuration (M = 10,000).
# usage: bash scripts/round_profile.sh rNN
R=${1:-r01}
cd "$GRAFT_REPO_ROOT"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$R.log 2>&1; tail -1 gpurun_out/bench_$R.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --compare "" > /dev/null 2>&1
for k in alc_incremental alc_explicit_dmma nn_pool; do
  f=incremental; [ "$k" = alc_explicit_dmma ] && f=explicit
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/prof_${k}_$R python scripts/profile_run.py --M 10000 --form $f > gpurun_out/ncu_${k}.log 2>&1
  tail -1 gpurun_out/ncu_${k}.log
done
