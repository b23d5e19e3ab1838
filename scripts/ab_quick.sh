#!/bin/bash
# quick A/B timing of the incremental kernel at C2 (10^4 locations) under env variants,
# then a parity subset. usage: bash scripts/ab_quick.sh "ENV1" "ENV2" ... (use "-" for default)
cd "$GRAFT_REPO_ROOT"
for env in "$@"; do
  [ "$env" = "-" ] && env=""
  echo "== $env"; env $env timeout 120 python scripts/profile_run.py --M 10000 --form incremental --reps 4 2>&1 | tail -1
done
timeout 900 python -m pytest tests -m gpu -x -q -k "${PYTEST_K:-alc_batch_vs_oracle or variants or north_star or smoke}" 2>&1 | tail -3
