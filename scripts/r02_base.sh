#!/bin/bash
# r02 baseline: bench line, launch list, ncu full of v2 + NN at the bench config
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02a.log 2>&1; tail -1 gpurun_out/bench_r02a.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02a.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --compare "" > /dev/null 2>&1
for k in alc_incremental_v2 nn_pool; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/prof_${k}_r02a python scripts/profile_run.py --M 10000 --form incremental > gpurun_out/ncu_${k}.log 2>&1
  tail -1 gpurun_out/ncu_${k}.log
done
