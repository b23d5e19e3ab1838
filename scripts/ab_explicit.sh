#!/bin/bash
# explicit (DMMA) form at C2: timing and DRAM / DMMA-pipe counters under env variants
cd "$GRAFT_REPO_ROOT"
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct"
for env in "$@"; do
  [ "$env" = "-" ] && env=""
  echo "== $env"; env $env timeout 300 python scripts/profile_run.py --M 10000 --form explicit --reps 2 2>&1 | tail -1
  env $env timeout 600 ncu --metrics $M -k regex:alc_explicit_dmma -c 1 --csv python scripts/profile_run.py --M 10000 --form explicit 2>/dev/null | grep -v "^==" | cut -d, -f10- | tail -8
done
timeout 900 python -m pytest tests -m gpu -x -q -k "${PYTEST_K:-explicit}" 2>&1 | tail -3
