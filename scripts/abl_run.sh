cd "$GRAFT_REPO_ROOT"
for a in 1 2 4 7; do echo "abl=$a $(python scripts/profile_run.py --M 10000 --form incremental --reps 3 --lib paper_1310_5182_b200/liblagp_abl$a.so 2>&1 | tail -1)"; done
echo "base $(python scripts/profile_run.py --M 10000 --form incremental --reps 3 2>&1 | tail -1)"
