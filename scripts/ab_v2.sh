#!/bin/bash
# A/B of the incremental kernel's switches at C2 (10^4 locations), then the GPU parity tests.
# usage: bash scripts/ab_v2.sh [pytest -k expr]
cd "$GRAFT_REPO_ROOT"
for env in "" "LAGP_V2_SFIRST=1" "LAGP_V2_CPT=4" "LAGP_V2_NOSTAGGER=1"; do
  echo "== $env"; env $env timeout 120 python scripts/profile_run.py --M 10000 --form incremental --reps 3 2>&1 | tail -1
done
K=${1:-"incremental or variants or north_star or smoke or fullsize"}
timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" 2>&1 | tail -15
