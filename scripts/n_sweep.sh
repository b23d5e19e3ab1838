cd "$GRAFT_REPO_ROOT"
for n in 7 10 20 30 40 50 60; do echo "n=$n $(python scripts/profile_run.py --M 10000 --form incremental --reps 3 --n $n 2>&1 | tail -1)"; done
